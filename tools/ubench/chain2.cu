// Where does a one-warp triangular-solve step lose time?  Per step (slice):
//   base: W ring gathers (slots + values in shared memory, LDS.128) -> DFMA chain -> STS -> __syncwarp
//   +stg: a scattered 8-byte global store per lane
//   +cpa: cp.async of a 2 KB record 15 steps ahead + commit + wait_group 15
#include <cstdio>
#include <cuda_runtime.h>

constexpr int W = 4;
template <int MODE>
__global__ void k(double *out, double *gsc, const unsigned char *rec, long long *t, int n) {
  __shared__ double ring[1024];
  __shared__ __align__(16) unsigned short slots[16][32][8];
  __shared__ __align__(16) double vals[16][32][W];
  __shared__ __align__(16) unsigned char stage[16][1024];
  const int lane = threadIdx.x;
  for (int i = lane; i < 1024; i += 32) ring[i] = 1e-3 * i;
  for (int s = 0; s < 16; ++s)
    for (int e = 0; e < 8; ++e) slots[s][lane][e] = (unsigned short)((((s + 15) % 16) * 32 + ((lane * 7 + e * 5) & 31)) & 1023);
  for (int s = 0; s < 16; ++s)
    for (int e = 0; e < W; ++e) vals[s][lane][e] = 1e-4 * (e + 1);
  __syncwarp();
  long long t0 = clock64();
  for (int it = 0; it < n; ++it) {
    const int s = it & 15;
    if (MODE & 2) {
      unsigned char *sp = stage[(it + 15) & 15];
      const unsigned char *src = rec + ((size_t)(it + 15) % 4096) * 1024;
      for (int o = lane * 16; o < 1024; o += 512) {
        unsigned d = (unsigned)__cvta_generic_to_shared(sp + o);
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(src + o) : "memory");
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
      asm volatile("cp.async.wait_group 15;" ::: "memory");
      __syncwarp();
    }
    const uint4 c = *reinterpret_cast<const uint4 *>(&slots[s][lane][0]);
    const double2 v01 = *reinterpret_cast<const double2 *>(&vals[s][lane][0]);
    const double2 v23 = *reinterpret_cast<const double2 *>(&vals[s][lane][2]);
    double a0 = 1.0 + (MODE & 2 ? (double)stage[it & 15][lane] * 1e-9 : 0.0), a1 = 0, a2 = 0, a3 = 0;
    a0 -= v01.x * ring[c.x & 0xffff];
    a1 -= v01.y * ring[c.x >> 16];
    a2 -= v23.x * ring[c.y & 0xffff];
    a3 -= v23.y * ring[c.y >> 16];
    const double acc = ((a0 + a1) + (a2 + a3)) * 0.999;
    ring[(s * 32 + lane) & 2047] = acc;
    __syncwarp();
    if (MODE & 1) gsc[((size_t)it * 977 + lane * 4099) & ((1 << 22) - 1)] = acc;
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");
  long long t1 = clock64();
  out[lane] = ring[lane];
  if (lane == 0) t[MODE] = t1 - t0;
}

int main() {
  double *o, *g; unsigned char *rec; long long *t, h[4];
  cudaMalloc(&o, 4096); cudaMalloc(&g, (1 << 22) * 8); cudaMalloc(&rec, 4096 * 2048); cudaMalloc(&t, 64);
  cudaMemset(rec, 0, 4096 * 2048);
  const int n = 20000;
  k<0><<<1, 32>>>(o, g, rec, t, n); k<0><<<1, 32>>>(o, g, rec, t, n);
  k<1><<<1, 32>>>(o, g, rec, t, n); k<1><<<1, 32>>>(o, g, rec, t, n);
  k<2><<<1, 32>>>(o, g, rec, t, n); k<2><<<1, 32>>>(o, g, rec, t, n);
  k<3><<<1, 32>>>(o, g, rec, t, n); k<3><<<1, 32>>>(o, g, rec, t, n);
  cudaDeviceSynchronize();
  cudaMemcpy(h, t, 32, cudaMemcpyDeviceToHost);
  const char *nm[] = {"base", "+stg", "+cp.async", "+both"};
  for (int m = 0; m < 4; ++m) printf("%-10s %.1f cycles per step\n", nm[m], (double)h[m] / n);
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
