// Cost of issuing global loads on a barrier-paced critical path.
// 16 warps pass `nlev` barriers; at level v warp v % 16 consumes 10 values it
// loaded 16 levels earlier and issues the next 10 loads (each to a new line,
// DRAM miss) with the load flavour of `mode`.
#include <cstdio>
#include <cuda_runtime.h>

template <int MODE>
__device__ inline double ld(const double *q) {
  double v;
  if (MODE == 1) asm volatile("ld.global.f64 %0, [%1];" : "=d"(v) : "l"(q));
  else if (MODE == 2) asm volatile("ld.global.nc.f64 %0, [%1];" : "=d"(v) : "l"(q));
  else if (MODE == 3) asm volatile("ld.global.cg.f64 %0, [%1];" : "=d"(v) : "l"(q));
  else if (MODE == 4) asm volatile("ld.global.cs.f64 %0, [%1];" : "=d"(v) : "l"(q));
  else if (MODE == 5) asm volatile("ld.global.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(q));
  else if (MODE == 6) asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(q));
  else if (MODE == 7) asm volatile("ld.relaxed.gpu.global.f64 %0, [%1];" : "=d"(v) : "l"(q));
  else v = 1.0;
  return v;
}

template <int MODE>
__global__ void __launch_bounds__(512, 1) k(const double *__restrict__ src, double *out, long long *t, int nlev) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double v[10], acc = 0;
  for (int u = 0; u < 10; ++u) v[u] = 0;
  const double *p = src + (size_t)blockIdx.x * (1 << 22) + lane;
  int k = 0;
  long long t0 = clock64();
  long long tl = 0;
  for (int lv = 0; lv < nlev; ++lv) {
    if ((lv & 15) == warp) {
      for (int u = 0; u < 10; ++u) acc += v[u];
      const double *q = p + (size_t)(k++) * 8192 + warp * 32 * 64;   // new lines every time (DRAM miss)
      long long a = clock64();
#pragma unroll
      for (int u = 0; u < 10; ++u) v[u] = ld<MODE>(q + u * 32 * 4);
      tl += clock64() - a;
    }
    asm volatile("bar.sync 1, 512;" ::: "memory");
  }
  long long t1 = clock64();
  out[blockIdx.x * 512 + threadIdx.x] = acc + v[0];
  if (threadIdx.x == 0 && blockIdx.x == 0) { t[2 * MODE] = t1 - t0; t[2 * MODE + 1] = tl; }
}

int main() {
  double *src, *out;
  long long *t, h[16];
  const int nb = 32;
  cudaMalloc(&src, (size_t)nb * (1 << 22) * 8 + (1 << 27));
  cudaMemset(src, 0, (size_t)nb * (1 << 22) * 8 + (1 << 27));
  cudaMalloc(&out, nb * 512 * 8);
  cudaMalloc(&t, 128);
  const int nlev = 2000;
  auto run = [&](auto kern) { kern<<<nb, 512>>>(src, out, t, nlev); kern<<<nb, 512>>>(src, out, t, nlev); cudaDeviceSynchronize(); };
  run(k<0>); run(k<1>); run(k<2>); run(k<3>); run(k<4>); run(k<5>); run(k<6>); run(k<7>);
  cudaMemcpy(h, t, 128, cudaMemcpyDeviceToHost);
  const char *nm[] = {"none", "ld.global", "ld.nc", "ld.cg", "ld.cs", "L1::no_allocate", "nc.L1::no_alloc", "relaxed.gpu"};
  for (int m = 0; m < 8; ++m)
    printf("%-16s %7.1f cycles per level, issue of 10 loads %7.1f cycles\n", nm[m], (double)h[2 * m] / nlev, (double)h[2 * m + 1] / (nlev / 16));
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
