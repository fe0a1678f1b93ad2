// Floor of the triangular-solve dependency chain on one warp: per step, W
// gathers from a shared-memory ring (slots of the previous step's results),
// a DFMA chain, a store of the step's result and __syncwarp.
#include <cstdio>
#include <cuda_runtime.h>

template <int W, int SYNC>
__global__ void k(double *out, long long *t, int n) {
  __shared__ double ring[2048];
  __shared__ unsigned short slots[32][32][W];
  const int lane = threadIdx.x;
  for (int i = lane; i < 2048; i += 32) ring[i] = 1e-3 * i;
  for (int s = 0; s < 32; ++s)
    for (int e = 0; e < W; ++e) slots[s][lane][e] = (unsigned short)((((s + 31) % 32) * 32 + ((lane * 7 + e * 5) & 31)) & 2047);
  __syncwarp();
  double vals[W];
  for (int e = 0; e < W; ++e) vals[e] = 1e-4 * (e + 1);
  long long t0 = clock64();
  for (int it = 0; it < n; ++it) {
    const int s = it & 31;
    double a0 = 1.0, a1 = 0, a2 = 0, a3 = 0;
#pragma unroll
    for (int e = 0; e < W; e += 4) {
      a0 -= vals[e] * ring[slots[s][lane][e]];
      if (e + 1 < W) a1 -= vals[e + 1] * ring[slots[s][lane][e + 1]];
      if (e + 2 < W) a2 -= vals[e + 2] * ring[slots[s][lane][e + 2]];
      if (e + 3 < W) a3 -= vals[e + 3] * ring[slots[s][lane][e + 3]];
    }
    const double acc = ((a0 + a1) + (a2 + a3)) * 0.999;
    ring[(s * 32 + lane) & 4095] = acc;
    if (SYNC) __syncwarp();
  }
  long long t1 = clock64();
  out[lane] = ring[lane];
  if (lane == 0) t[0] = t1 - t0;
}

int main() {
  double *o; long long *t, h;
  cudaMalloc(&o, 4096); cudaMalloc(&t, 64);
  const int n = 20000;
  auto run = [&](auto kern, const char *nm) {
    kern<<<1, 32>>>(o, t, n); kern<<<1, 32>>>(o, t, n); cudaDeviceSynchronize();
    cudaMemcpy(&h, t, 8, cudaMemcpyDeviceToHost);
    printf("%-16s %.1f cycles per step\n", nm, (double)h / n);
  };
  run(k<4, 1>, "W=4 syncwarp");
  run(k<10, 1>, "W=10 syncwarp");
  run(k<4, 0>, "W=4 no sync");
  run(k<10, 0>, "W=10 no sync");
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
