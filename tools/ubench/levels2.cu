// k_tri_reg level protocol vs the number of consumer warps NW (one record buffer per warp).
// Slice s -> warp s % NW, level s / K.  A warp arrives (bar.arrive) at every level before
// its next slice's right after its own slice, syncs (bar.sync) on the level before its next
// slice, and never arrives more than 15 levels past the last level it saw complete (it syncs
// instead), so 15 rotating barrier ids never alias for any NW.  Per slice: W = 10 ring
// gathers + DFMA chain + STS, then a scattered 8-byte global store, an L2 bulk prefetch
// 6 slices ahead and 8 x 16-byte record loads for its next slice (consumed there).
#include <cstdio>
#include <cuda_runtime.h>

constexpr int W = 10, R = 4096;

template <int NW> __device__ inline void arrive(int v) { asm volatile("bar.arrive %0, %1;" ::"r"(1 + v % 15), "n"(32 * NW) : "memory"); }
template <int NW> __device__ inline void sync(int v) { asm volatile("bar.sync %0, %1;" ::"r"(1 + v % 15), "n"(32 * NW) : "memory"); }

template <int NW, int LD>
__global__ void __launch_bounds__(32 * NW, 1) k(const uint4 *__restrict__ rec, double *gout, long long *t, int ns, int K) {
  __shared__ double ring[R];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < R; i += blockDim.x) ring[i] = 1e-3 * (i & 7);
  __syncthreads();
  const uint4 *rb = rec + (size_t)blockIdx.x * ns * 8 * 32;
  uint4 q[8];
  for (int j = 0; j < 8; ++j) q[j] = make_uint4(0, 0, 0, 0);
  const int nlev = (ns + K - 1) / K;
  int cur = 0, known = -1;   // cur: next level to arrive at; known: last level seen complete
  auto step = [&](int u) {   // pass level u without a slice in it
    if (NW > 15 && u - known >= 15) { sync<NW>(u); known = u; }   // instance u - 15 of this id must be complete
    else arrive<NW>(u);
  };
  long long t0 = clock64();
  for (int s = warp; s < ns; s += NW) {
    const int lv = s / K;
    for (; cur < lv - 1; ++cur) step(cur);
    if (cur < lv) { sync<NW>(cur); known = cur; ++cur; }
    const int pb = (lv > 0 ? (lv - 1) * K : 0) * 32;
    double acc = 1.0 + (LD ? (double)(q[0].x & 1) : 0.0), a1 = 0, a2 = 0, a3 = 0;
#pragma unroll
    for (int e = 0; e < W; e += 4) {
      auto sl = [&](int f) { return (pb + (lane * 3 + f * 7) % (32 * K)) & (R - 1); };
      acc -= 0.5 * ring[sl(e)];
      if (e + 1 < W) a1 -= 0.25 * ring[sl(e + 1)];
      if (e + 2 < W) a2 -= 0.125 * ring[sl(e + 2)];
      if (e + 3 < W) a3 -= 0.0625 * ring[sl(e + 3)];
    }
    acc = (acc + a1) + (a2 + a3);
    ring[(s * 32 + lane) & (R - 1)] = acc;
    const int nxt = s + NW < ns ? (s + NW) / K : nlev;
    for (; cur < nxt - 1 && (NW <= 15 || cur - known < 15); ++cur) arrive<NW>(cur);   // non-blocking part first
    gout[((size_t)blockIdx.x << 20) + (((size_t)s * 977 + lane * 4099) & ((1 << 20) - 1))] = acc;
    if (LD) {
      const int sp = s + 6 * NW < ns ? s + 6 * NW : s;
      if (lane == 0) asm volatile("cp.async.bulk.prefetch.L2.global [%0], 4096;" ::"l"(rb + (size_t)sp * 8 * 32) : "memory");
      const uint4 *p = rb + (size_t)(s + NW < ns ? s + NW : s) * 8 * 32 + lane;
#pragma unroll
      for (int j = 0; j < 8; ++j) q[j] = __ldg(p + 32 * j);
    }
    for (; cur < nxt - 1; ++cur) step(cur);
  }
  for (; cur < nlev; ++cur) arrive<NW>(cur);
  long long t1 = clock64();
  if (lane == 0 && warp == 0 && blockIdx.x == 0) t[0] = t1 - t0;
  unsigned x = 0;
  for (int j = 0; j < 8; ++j) x ^= q[j].x ^ q[j].w;
  if (x == 12345) gout[threadIdx.x] = x;
}

int main() {
  const int nb = 32, ns = 6000;
  uint4 *rec; double *g; long long *t, h;
  cudaMalloc(&rec, (size_t)nb * ns * 8 * 32 * 16);
  cudaMemset(rec, 0, (size_t)nb * ns * 8 * 32 * 16);
  cudaMalloc(&g, (size_t)nb << 23);
  cudaMalloc(&t, 64);
  auto run = [&](auto kern, int nw, int ld) {
    printf("NW=%2d %s", nw, ld ? "loads   " : "no loads");
    for (int K : {1, 2, 4, 6, 8, 12}) {
      kern<<<nb, 32 * nw>>>(rec, g, t, ns, K);
      kern<<<nb, 32 * nw>>>(rec, g, t, ns, K);
      cudaDeviceSynchronize();
      cudaMemcpy(&h, t, 8, cudaMemcpyDeviceToHost);
      printf("  K=%2d %6.1f", K, (double)h / ((ns + K - 1) / K));
    }
    printf("  cycles/level\n");
  };
  run(k<15, 0>, 15, 0); run(k<15, 1>, 15, 1);
  run(k<23, 0>, 23, 0); run(k<23, 1>, 23, 1);
  run(k<31, 0>, 31, 0); run(k<31, 1>, 31, 1);
  run(k<8, 0>, 8, 0); run(k<8, 1>, 8, 1);
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
