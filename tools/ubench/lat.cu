// Microbenchmark: dependent DFMA latency, dependent LDS latency, named barrier cost (B200).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double *out, long long *t, int n) {
  __shared__ int sidx[1024];
  __shared__ double sval[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) { sidx[i] = (i * 97 + 13) & 1023; sval[i] = 1.0 + i * 1e-6; }
  __syncthreads();
  double a = out[threadIdx.x], b = 1.0000001, c = 1e-9;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) a = fma(a, b, c);
  long long t1 = clock64();
  int p = threadIdx.x & 1023;
  for (int i = 0; i < n; ++i) p = sidx[p];
  long long t2 = clock64();
  double s = 0;
  for (int i = 0; i < n; ++i) { s += sval[p]; p = (p + 1) & 1023; }
  long long t3 = clock64();
  for (int i = 0; i < n; ++i) asm volatile("bar.sync 1, 256;");
  long long t4 = clock64();
  for (int i = 0; i < n; ++i) __syncthreads();
  long long t5 = clock64();
  out[threadIdx.x] = a + p + s;
  if (threadIdx.x == 0) { t[0] = t1 - t0; t[1] = t2 - t1; t[2] = t3 - t2; t[3] = t4 - t3; t[4] = t5 - t4; }
}
int main() {
  double *o; long long *t, h[5];
  cudaMalloc(&o, 4096 * 8); cudaMemset(o, 0, 4096 * 8); cudaMalloc(&t, 64);
  int n = 4096;
  k<<<1, 256>>>(o, t, n); cudaDeviceSynchronize();
  k<<<1, 256>>>(o, t, n); cudaMemcpy(h, t, 40, cudaMemcpyDeviceToHost);
  printf("DFMA dep latency %.1f cyc, LDS dep latency %.1f cyc, LDS+DADD dep %.1f, bar.sync(256) %.1f, syncthreads %.1f\n",
         (double)h[0] / n, (double)h[1] / n, (double)h[2] / n, (double)h[3] / n, (double)h[4] / n);
  return 0;
}
