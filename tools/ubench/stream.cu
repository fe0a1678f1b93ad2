// Microbenchmarks for the trisolve redesign (B200):
//  (1) per-SM streaming bandwidth of 1D bulk copies (TMA, UBLKCP) into a smem ring,
//      with and without the consumers reading the bytes back (LDS), and of direct
//      LDG.128 streaming, at 1 / 32 / 64 / 148 CTAs;
//  (2) hand-off latency between two warps of one CTA through a shared-memory flag,
//      between two CTAs of a cluster through DSMEM, and through global memory.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s line %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

__device__ inline unsigned su32(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ inline void mb_init(uint64_t *b, unsigned c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(c) : "memory"); }
__device__ inline void mb_tx(uint64_t *b, unsigned by) { asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(by) : "memory"); }
__device__ inline void mb_arrive(uint64_t *b) { asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory"); }
__device__ inline void mb_wait(uint64_t *b, unsigned par) {
  asm volatile("{\n\t.reg .pred P1;\nW1:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t@P1 bra D1;\n\tbra W1;\nD1:\n\t}" ::"r"(su32(b)), "r"(par) : "memory");
}
__device__ inline void bulk(void *d, const void *s, unsigned by, uint64_t *b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su32(d)), "l"(s), "r"(by), "r"(su32(b)) : "memory");
}

constexpr int CH = 16384, NST = 6, NCW = 8;
// per CTA: stream `bytes` starting at src + blockIdx.x * bytes
__global__ void __launch_bounds__(32 * (NCW + 1), 1) k_tma(const char *src, size_t bytes, int consume, double *out) {
  extern __shared__ __align__(128) unsigned char sm[];
  uint64_t *full = reinterpret_cast<uint64_t *>(sm + NST * CH), *empty = full + NST;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) { for (int i = 0; i < NST; ++i) { mb_init(&full[i], 1); mb_init(&empty[i], NCW); } asm volatile("fence.mbarrier_init.release.cluster;"); }
  __syncthreads();
  const char *p = src + (size_t)blockIdx.x * bytes;
  const int nk = (int)(bytes / CH);
  if (warp == NCW) {
    if (lane) return;
    for (int k = 0; k < nk; ++k) {
      const int s = k % NST;
      if (k >= NST) mb_wait(&empty[s], ((k / NST) - 1) & 1);
      mb_tx(&full[s], CH);
      bulk(sm + s * CH, p + (size_t)k * CH, CH, &full[s]);
    }
    return;
  }
  double acc = 0;
  for (int k = 0; k < nk; ++k) {
    const int s = k % NST;
    mb_wait(&full[s], (k / NST) & 1);
    if (consume) {
      const double2 *q = reinterpret_cast<const double2 *>(sm + s * CH);
#pragma unroll 4
      for (int i = threadIdx.x; i < CH / 16; i += 32 * NCW) { double2 v = q[i]; acc += v.x + v.y; }
    }
    __syncwarp();
    if (lane == 0) mb_arrive(&empty[s]);
  }
  if (acc == 12345.678) out[0] = acc;
}

template <int NW>
__global__ void __launch_bounds__(32 * NW, 1) k_ldg(const char *src, size_t bytes, double *out) {
  const double2 *p = reinterpret_cast<const double2 *>(src + (size_t)blockIdx.x * bytes);
  const size_t n = bytes / 16;
  double a0 = 0, a1 = 0;
  size_t i = threadIdx.x;
  for (; i + 7 * 32 * NW < n; i += 8 * 32 * NW) {
    double2 v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = __ldcs(p + i + u * 32 * NW);
#pragma unroll
    for (int u = 0; u < 8; ++u) { a0 += v[u].x; a1 += v[u].y; }
  }
  if (a0 + a1 == 12345.678) out[0] = a0;
}

// ping-pong between warp 0 and warp 1 (lane 0) through a smem flag
__global__ void k_pp_smem(long long *t, int n, int mode) {
  __shared__ volatile int f[64];
  if (threadIdx.x == 0) { f[0] = 0; f[32] = 0; }
  __syncthreads();
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) != 0 || w > 1) return;
  long long t0 = clock64();
  for (int i = 1; i <= n; ++i) {
    if (w == 0) {
      if (mode == 0) { f[0] = i; while (f[32] != i) {} }
      else {
        asm volatile("st.release.cta.shared.u32 [%0], %1;" ::"r"(su32((const void *)&f[0])), "r"(i) : "memory");
        int v; do { asm volatile("ld.acquire.cta.shared.u32 %0, [%1];" : "=r"(v) : "r"(su32((const void *)&f[32])) : "memory"); } while (v != i);
      }
    } else {
      if (mode == 0) { while (f[0] != i) {} f[32] = i; }
      else {
        int v; do { asm volatile("ld.acquire.cta.shared.u32 %0, [%1];" : "=r"(v) : "r"(su32((const void *)&f[0])) : "memory"); } while (v != i);
        asm volatile("st.release.cta.shared.u32 [%0], %1;" ::"r"(su32((const void *)&f[32])), "r"(i) : "memory");
      }
    }
  }
  if (w == 0) t[0] = clock64() - t0;
}

// ping-pong between CTA 0 and CTA 1 of a cluster through DSMEM: each waits on its own smem flag
__global__ void __cluster_dims__(2, 1, 1) k_pp_dsmem(long long *t, int n) {
  __shared__ int f;
  unsigned r; asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  if (threadIdx.x == 0) f = 0;
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  if (threadIdx.x == 0) {
    unsigned mine = su32(&f), peer;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(peer) : "r"(mine), "r"(r ^ 1u));
    long long t0 = clock64();
    for (int i = 1; i <= n; ++i) {
      if (r == 0) {
        asm volatile("st.release.cluster.shared::cluster.u32 [%0], %1;" ::"r"(peer), "r"(i) : "memory");
        int v; do { asm volatile("ld.acquire.cluster.shared::cta.u32 %0, [%1];" : "=r"(v) : "r"(mine) : "memory"); } while (v != i);
      } else {
        int v; do { asm volatile("ld.acquire.cluster.shared::cta.u32 %0, [%1];" : "=r"(v) : "r"(mine) : "memory"); } while (v != i);
        asm volatile("st.release.cluster.shared::cluster.u32 [%0], %1;" ::"r"(peer), "r"(i) : "memory");
      }
    }
    if (r == 0) t[1] = clock64() - t0;
  }
  __syncwarp();
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

__global__ void k_pp_gmem(int *f, long long *t, int n) {
  if (threadIdx.x) return;
  const int b = blockIdx.x;
  long long t0 = clock64();
  for (int i = 1; i <= n; ++i) {
    if (b == 0) {
      asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(f), "r"(i) : "memory");
      int v; do { asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(f + 32) : "memory"); } while (v != i);
    } else {
      int v; do { asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(f) : "memory"); } while (v != i);
      asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(f + 32), "r"(i) : "memory");
    }
  }
  if (b == 0) t[2] = clock64() - t0;
}

int main() {
  setvbuf(stdout, NULL, _IONBF, 0);
  const size_t per = 32u << 20;        // 32 MB per CTA
  const int grids[] = {1, 8, 32, 64, 148};
  char *buf; double *o; long long *t; int *f;
  CK(cudaMalloc(&buf, per * 148));
  CK(cudaMemset(buf, 1, per * 148));
  CK(cudaMalloc(&o, 64)); CK(cudaMalloc(&t, 64)); CK(cudaMalloc(&f, 1024));
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const int smem = NST * CH + 2 * NST * 8;
  CK(cudaFuncSetAttribute(k_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int g : grids) {
    for (int mode = 0; mode < 4; ++mode) {
      float best = 1e30f;
      for (int rep = 0; rep < 3; ++rep) {
        cudaEventRecord(e0);
        if (mode == 0) k_tma<<<g, 32 * (NCW + 1), smem>>>(buf, per, 0, o);
        else if (mode == 1) k_tma<<<g, 32 * (NCW + 1), smem>>>(buf, per, 1, o);
        else if (mode == 2) k_ldg<8><<<g, 256>>>(buf, per, o);
        else k_ldg<32><<<g, 1024>>>(buf, per, o);
        cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
        float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
      }
      const char *nm[] = {"tma only", "tma+lds", "ldg 8w", "ldg 32w"};
      printf("grid %3d %-9s: %8.1f GB/s total, %6.1f GB/s per CTA\n", g, nm[mode], per * g / best / 1e6, per / best / 1e6);
    }
  }
  long long h[3];
  const int n = 10000;
  for (int mode = 0; mode < 2; ++mode) {
    k_pp_smem<<<1, 64>>>(t, n, mode); CK(cudaDeviceSynchronize());
    cudaMemcpy(h, t, 8, cudaMemcpyDeviceToHost);
    printf("smem flag ping-pong (%s): %.1f cycles per one-way hand-off\n", mode ? "release/acquire" : "volatile", (double)h[0] / n / 2);
  }
  k_pp_dsmem<<<2, 32>>>(t, n); CK(cudaDeviceSynchronize());
  cudaMemcpy(h, t, 16, cudaMemcpyDeviceToHost);
  printf("dsmem ping-pong: %.1f cycles per one-way hand-off\n", (double)h[1] / n / 2);
  cudaMemset(f, 0, 1024);
  k_pp_gmem<<<2, 32>>>(f, t, n); CK(cudaDeviceSynchronize());
  cudaMemcpy(h, t, 24, cudaMemcpyDeviceToHost);
  printf("gmem ping-pong: %.1f cycles per one-way hand-off\n", (double)h[2] / n / 2);
  printf("sm clock attr %d kHz\n", clk);
  return 0;
}
