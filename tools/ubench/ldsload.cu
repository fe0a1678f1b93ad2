// Does shared-memory gather latency grow when other warps of the SM stream global loads?
// Warp 0 times a batch of 10 independent 8-byte LDS gathers (random slots of a
// 128 KB ring) followed by their use; warps 1..15 stream LDG.128 (mode 1) or idle (mode 0).
#include <cstdio>
#include <cuda_runtime.h>

__global__ void __launch_bounds__(512, 1) k(const double2 *__restrict__ src, double *out, long long *t, int mode, int reps) {
  extern __shared__ double ring[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 16384; i += blockDim.x) ring[i] = i * 1e-3;
  __syncthreads();
  volatile __shared__ int stop;
  if (threadIdx.x == 0) stop = 0;
  __syncthreads();
  if (warp == 0) {
    unsigned idx[10];
    unsigned seed = 12345u + lane * 7919u;
    double acc = 0;
    long long tot = 0;
    for (int r = 0; r < reps; ++r) {
      for (int e = 0; e < 10; ++e) { seed = seed * 1664525u + 1013904223u; idx[e] = (seed >> 8) & 16383; }
      __syncwarp();
      long long a = clock64();
      double v[10];
#pragma unroll
      for (int e = 0; e < 10; ++e) v[e] = ring[idx[e]];
      double s0 = 0, s1 = 0;
#pragma unroll
      for (int e = 0; e < 10; e += 2) { s0 += v[e]; s1 += v[e + 1]; }
      acc += s0 + s1;
      long long b = clock64() + (acc == -1.0 ? 1 : 0);
      tot += b - a;
      for (int w = 0; w < 50; ++w) __nanosleep(20);
    }
    if (lane == 0) { t[mode] = tot / reps; }
    out[lane] = acc;
    if (lane == 0) stop = 1;
  } else if (mode == 1) {
    const double2 *p = src + (size_t)blockIdx.x * (1 << 21) + (warp - 1) * 32 + lane;
    double s = 0;
    for (int it = 0; !stop && it < 100000; ++it) {
      double2 v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = __ldg(p + ((size_t)(it * 8 + u) * 480) % ((1 << 21) - 512));
#pragma unroll
      for (int u = 0; u < 8; ++u) s += v[u].x;
    }
    out[threadIdx.x + 32] = s;
  }
}

int main() {
  double2 *src; double *out; long long *t, h[2] = {0, 0};
  cudaMalloc(&src, (size_t)32 * (1 << 21) * 16);
  cudaMemset(src, 0, (size_t)32 * (1 << 21) * 16);
  cudaMalloc(&out, 4096 * 8); cudaMalloc(&t, 16);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 131072);
  for (int mode = 0; mode < 2; ++mode) {
    k<<<32, 512, 131072>>>(src, out, t, mode, 2000);
    printf("launch %d: %s\n", mode, cudaGetErrorString(cudaGetLastError()));
    printf("sync %d: %s\n", mode, cudaGetErrorString(cudaDeviceSynchronize()));
  }
  cudaMemcpy(h, t, 16, cudaMemcpyDeviceToHost);
  printf("10 LDS gathers + use: %lld cycles idle SM, %lld cycles with 15 warps streaming LDG.128\n", h[0], h[1]);
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
