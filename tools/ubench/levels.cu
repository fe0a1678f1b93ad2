// Cost of one level of the k_tri_reg protocol as a function of the slices per level.
// 15 consumer warps; slice s belongs to warp s % 15 and to level s / K.  A slice:
// (sync on the previous level's barrier if this warp has a slice there) -> W = 10
// ring gathers (LDS.64) of the previous level's outputs -> 4-way DFMA chain -> STS
// -> arrive on its level's barrier, then (MODE bit 0) 8 x 16-byte record loads for
// its next slice (DRAM/L2 stream) and (bit 1) a scattered 8-byte global store;
// bit 2: all lanes gather the same address (no bank conflicts).
// One CTA per SM on `nb` SMs, like the level-0 launch (32 blocks).
#include <cstdio>
#include <cuda_runtime.h>

constexpr int NW = 15, W = 10, R = 4096;

__device__ inline void arrive(int v) { asm volatile("bar.arrive %0, %1;" ::"r"(1 + v % 15), "n"(32 * NW) : "memory"); }
__device__ inline void sync(int v) { asm volatile("bar.sync %0, %1;" ::"r"(1 + v % 15), "n"(32 * NW) : "memory"); }

template <int MODE>
__global__ void __launch_bounds__(32 * NW, 1) k(const uint4 *__restrict__ rec, double *gout, long long *t, int ns, int K) {
  extern __shared__ __align__(128) unsigned char dsm[];
  double *ring = reinterpret_cast<double *>(dsm);
  uint4 *stage = reinterpret_cast<uint4 *>(dsm + R * 8);        // [warp][2][8][32] uint4 (cp.async records)
  __shared__ __align__(8) unsigned long long mb[16];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  constexpr unsigned E = (1u << 20) - 1;   // fixed expected count; the first slice of a level tops it up
  if (threadIdx.x < 16) asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(&mb[threadIdx.x])), "r"(E) : "memory");
  int done = -1;
  for (int i = threadIdx.x; i < R; i += blockDim.x) ring[i] = 1e-3 * (i & 7);
  __syncthreads();
  const uint4 *rb = rec + (size_t)blockIdx.x * ns * 8 * 32;
  uint4 q[8];
  for (int j = 0; j < 8; ++j) q[j] = make_uint4(0, 0, 0, 0);
  int cur = 0;
  long long t0 = clock64();
  for (int s = warp; s < ns; s += NW) {
    const int lv = s / K;
    if (MODE & 1024) {                                        // bit 10: just-in-time loads of this slice (L1-prefetched a slice earlier)
      const uint4 *p = rb + (size_t)s * 8 * 32 + lane;
#pragma unroll
      for (int j = 0; j < 8; ++j) q[j] = __ldg(p + 32 * j);
    }
    if (MODE & 256) {                                         // bit 8: record of this slice from its cp.async stage
      asm volatile("cp.async.wait_group 1;" ::: "memory");
      __syncwarp();
      const uint4 *st = stage + ((size_t)(warp * 2 + ((s / NW) & 1)) * 8) * 32 + lane;
#pragma unroll
      for (int j = 0; j < 8; ++j) q[j] = st[32 * j];
    }
    if (MODE & 64) {                                          // bit 6: mbarrier per level, only the producers arrive
      if (lv > 0 && done < lv - 1) {
        const unsigned a = (unsigned)__cvta_generic_to_shared(&mb[(lv - 1) & 15]), par = ((lv - 1) >> 4) & 1;
        unsigned ok = 0;
        while (!ok)
          asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                       : "=r"(ok) : "r"(a), "r"(par) : "memory");
        done = lv - 1;
      }
    } else {
      for (; cur < lv - 1; ++cur) arrive(cur);
      if (cur < lv) { sync(cur); ++cur; }
    }
    const int pb = (lv > 0 ? (lv - 1) * K : 0) * 32;   // previous level's outputs
    double acc = 1.0 + ((MODE & 512) ? 0.0 : (double)(q[0].x & 1)), a1 = 0, a2 = 0, a3 = 0;   // bit 9: loads never read in the loop
#pragma unroll
    for (int e = 0; e < W; e += 4) {
      auto sl = [&](int f) {
        const int o = (MODE & 4) ? 0 : (lane * 3 + f * 7) % (32 * K);
        return (pb + o) & (R - 1);
      };
      acc -= 0.5 * ring[sl(e)];
      if (e + 1 < W) a1 -= 0.25 * ring[sl(e + 1)];
      if (e + 2 < W) a2 -= 0.125 * ring[sl(e + 2)];
      if (e + 3 < W) a3 -= 0.0625 * ring[sl(e + 3)];
    }
    acc = (acc + a1) + (a2 + a3);
    ring[(s * 32 + lane) & (R - 1)] = acc;
    if (MODE & 64) {
      __syncwarp();
      if (lane == 0) {
        const int nl = min(K, ns - lv * K);
        const unsigned cnt = (s % K == 0) ? E - nl + 1 : 1;
        asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(&mb[lv & 15])), "r"(cnt) : "memory");
      }
    } else if (MODE & 32) {                                           // bit 5: arrive for every level before the next slice's now
      const int nxt = s + NW < ns ? (s + NW) / K : (ns + K - 1) / K;
      for (; cur < nxt - 1; ++cur) arrive(cur);
    } else if (s + NW >= ns || (s + NW) / K > lv + 1) { arrive(lv); cur = lv + 1; }
    if (MODE & 2) gout[((size_t)blockIdx.x << 20) + (((size_t)s * 977 + lane * 4099) & ((1 << 20) - 1))] = acc;
    if (MODE & 1) {
      const int sl = (MODE & 8) ? (s % (2 * NW)) : (s + 2 * NW < ns ? s + 2 * NW : s);   // bit 3: L1-resident records
      const uint4 *p = rb + (size_t)sl * 8 * 32 + lane;
      if (MODE & 128) {                                                                // bit 7: + L2 prefetch 6 slices ahead
        const int sp = s + 6 * NW < ns ? s + 6 * NW : s;
        if (lane == 0) asm volatile("cp.async.bulk.prefetch.L2.global [%0], 4096;" ::"l"(rb + (size_t)sp * 8 * 32) : "memory");
      }
      if (MODE & 1024) {
        const uint4 *pn = rb + (size_t)(s + NW < ns ? s + NW : s) * 8 * 32 + lane;
#pragma unroll
        for (int j = 0; j < 8; ++j) asm volatile("prefetch.global.L1 [%0];" ::"l"(pn + 32 * j) : "memory");
      } else if (MODE & 16) {                                                          // bit 4: L2 prefetch only
        if (lane == 0) asm volatile("cp.async.bulk.prefetch.L2.global [%0], 4096;" ::"l"(p) : "memory");
      } else if (MODE & 256) {
        __syncwarp();
        uint4 *st = stage + ((size_t)(warp * 2 + ((s / NW) & 1)) * 8) * 32 + lane;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const unsigned d = (unsigned)__cvta_generic_to_shared(st + 32 * j);
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(p + 32 * j) : "memory");
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
      } else {
#pragma unroll
        for (int j = 0; j < 8; ++j) q[j] = __ldg(p + 32 * j);
      }
    }
  }
  if (!(MODE & 64)) for (; cur < (ns + K - 1) / K; ++cur) arrive(cur);
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
  const size_t smem = R * 8 + (size_t)NW * 2 * 8 * 32 * 16;
  auto run = [&](auto kern, int mode) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const char *nm[] = {"base", "+ldg", "+stg", "+ldg+stg", "bcast", "bcast+ldg", "bcast+stg", "bcast+ldg+stg"};
    printf("%-14s%s%s%s%s%s%s%s%s", nm[mode & 7], mode & 8 ? " L1" : "", mode & 16 ? " pfL2" : "", mode & 32 ? " early" : "", mode & 64 ? " mbar" : "", mode & 128 ? " +pf" : "", mode & 256 ? " cp.async" : "", mode & 512 ? " unread" : "", mode & 1024 ? " L1pf+jit" : "");
    for (int K : {1, 2, 4, 6, 8}) {
      kern<<<nb, 32 * NW, smem>>>(rec, g, t, ns, K);
      kern<<<nb, 32 * NW, smem>>>(rec, g, t, ns, K);
      cudaDeviceSynchronize();
      cudaMemcpy(&h, t, 8, cudaMemcpyDeviceToHost);
      printf("  K=%d %6.1f", K, (double)h / ((ns + K - 1) / K));
    }
    printf("  cycles/level\n");
  };
  run(k<0>, 0); run(k<1>, 1); run(k<3>, 3); run(k<9>, 9); run(k<11>, 11);
  printf("L1 prefetch + just-in-time loads (bit 10):\n");
  run(k<1024 + 129>, 1024 + 129); run(k<1024 + 131>, 1024 + 131); run(k<1024 + 163>, 1024 + 163); run(k<1024 + 1>, 1024 + 1);
  printf("loads never consumed in the loop (bit 9):\n");
  run(k<512 + 129>, 512 + 129); run(k<512 + 131>, 512 + 131); run(k<512 + 163>, 512 + 163); run(k<512 + 1>, 512 + 1); run(k<512 + 33>, 512 + 33);
  printf("with L2 prefetch 6 slices ahead:\n");
  run(k<129>, 129); run(k<131>, 131); run(k<161>, 161); run(k<163>, 163); run(k<193>, 193); run(k<195>, 195);
  printf("cp.async staging:\n");
  run(k<257>, 257); run(k<259>, 259); run(k<385>, 385); run(k<387>, 387); run(k<419>, 419);
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
