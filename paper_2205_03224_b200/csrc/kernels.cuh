// sm_100a kernels of the GeMSLR solve path (arXiv 2205.03224).
//
// Every kernel is bandwidth- or latency-bound GEMV/SpMV-class work (<= 0.5
// flop/byte), so none uses tensor cores; they are written for coalesced
// 128-byte warp accesses, many loads in flight per thread, grids sized to the
// 148 SMs and deterministic (fixed-order) reductions.
//
//   k_spmv_sell     K1   y = A x / r = b - A x, SELL-32 (one warp per 32 rows)    Note N P:L58-61
//   k_trisolve      K4/K5/K9  level-scheduled L then U sweep per block; one CTA or
//                   one thread-block cluster per block, CTA/cluster barriers       Alg.2 l.2, l.9 P:L552,L561
//   k_ew            K6+K7  r_J = src_J - E_l z1 ; s = W_l^H r_J ; t = G_l s         Alg.2 l.3, l.7 P:L553,L558
//   k_waxpy         K8   r_J += W_l t
//   k_gs            K10-K12  CGS2 passes (multi-dot / update+dot / update+norm)
//   k_fgmres_col    Hessenberg column, Givens rotation, convergence flag (1 thread) P:L695-697
//   k_xupdate       K13  x += Z y
//   k_scale, k_perm K14  vector utilities
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace gemslr {

// Programmatic dependent launch (the FGMRES iteration's kernels are launched
// with cudaLaunchAttributeProgrammaticStreamSerialization): a kernel lets its
// successor's CTAs be scheduled at once and waits for its predecessor's
// completion (and memory flush) before reading anything it produced.  Both are
// no-ops for a normal launch.
__device__ inline void pdl_launch() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ inline void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }


constexpr int PIPE_SB_DEV = 30 * 1024;    // = PIPE_SB
constexpr int PIPE_NW_DEV = 8;            // = PIPE_NW

// ----------------------------------------------------------------- scalars
struct cd {
  double x, y;
};
__host__ __device__ inline cd operator+(cd a, cd b) { return {a.x + b.x, a.y + b.y}; }
__host__ __device__ inline cd operator-(cd a, cd b) { return {a.x - b.x, a.y - b.y}; }
__host__ __device__ inline cd operator-(cd a) { return {-a.x, -a.y}; }
__host__ __device__ inline cd operator*(cd a, cd b) { return {a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x}; }
__host__ __device__ inline cd operator*(double a, cd b) { return {a * b.x, a * b.y}; }
__host__ __device__ inline cd &operator+=(cd &a, cd b) { a.x += b.x; a.y += b.y; return a; }
__host__ __device__ inline cd &operator-=(cd &a, cd b) { a.x -= b.x; a.y -= b.y; return a; }
__host__ __device__ inline cd operator/(cd a, cd b) {
  // (a conj(b)) / |b|^2 — division by the U diagonal of complex ILU factors
  const double d = b.x * b.x + b.y * b.y;
  return {(a.x * b.x + a.y * b.y) / d, (a.y * b.x - a.x * b.y) / d};
}
__host__ __device__ inline double dconj(double a) { return a; }
__host__ __device__ inline cd dconj(cd a) { return {a.x, -a.y}; }
__host__ __device__ inline double dabs2(double a) { return a * a; }
__host__ __device__ inline double dabs2(cd a) { return a.x * a.x + a.y * a.y; }
template <typename T> __host__ __device__ inline T dzero();
template <> __host__ __device__ inline double dzero<double>() { return 0.0; }
template <> __host__ __device__ inline cd dzero<cd>() { return {0.0, 0.0}; }
__host__ __device__ inline double dscale(double a, double s) { return a * s; }
__host__ __device__ inline cd dscale(cd a, double s) { return {a.x * s, a.y * s}; }

__device__ inline double shfl_xor(double v, int m) { return __shfl_xor_sync(0xffffffffu, v, m); }
__device__ inline cd shfl_xor(cd v, int m) { return {__shfl_xor_sync(0xffffffffu, v.x, m), __shfl_xor_sync(0xffffffffu, v.y, m)}; }
template <typename T>
__device__ inline T warp_sum(T v) {
#pragma unroll
  for (int m = 16; m > 0; m >>= 1) v += shfl_xor(v, m);
  return v;
}

// L2-coherent loads (bypass L1) for vectors written by other CTAs of a cluster
__device__ inline double ld_cg(const double *p) { return __ldcg(p); }
__device__ inline cd ld_cg(const cd *p) {
  double2 v = __ldcg(reinterpret_cast<const double2 *>(p));
  return {v.x, v.y};
}
__device__ inline double ld_nc(const double *p) { return __ldg(p); }
__device__ inline double2 ld_na(const double2 *p) {             // read-only, no L1 allocation
  double2 v;
  asm("ld.global.nc.L1::no_allocate.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
  return v;
}
__device__ inline uint4 ld_na(const uint4 *p) {
  uint4 v;
  asm("ld.global.nc.L1::no_allocate.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
  return v;
}
__device__ inline cd ld_nc(const cd *p) {
  double2 v = __ldg(reinterpret_cast<const double2 *>(p));
  return {v.x, v.y};
}

__device__ inline unsigned cluster_ctarank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ inline void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// ----------------------------------------------------------------- K1 SpMV
// SELL-32: slice s holds rows 32s..32s+31; entry e of lane r at off[s] + 32e + r;
// padding has col = -1.  mode 0: y = A x ; mode 1: y = b - A x.
// Columns c >= nloc refer to the halo buffer xh (values received from the
// owners of exterior columns, Note N P:L59-61); one GPU has no halo.
template <typename T, bool HALO>
__global__ void __launch_bounds__(256) k_spmv_sell(int64_t n, int64_t nslices, const int64_t *__restrict__ off,
                                                   const int32_t *__restrict__ col, const T *__restrict__ val,
                                                   const T *__restrict__ x, const T *__restrict__ xh, T *__restrict__ y,
                                                   int mode, const T *__restrict__ b, const int *__restrict__ done) {
  if (done && *done) return;
  const int64_t s = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (s >= nslices) return;
  const int lane = threadIdx.x & 31;
  const int64_t o = off[s];
  const int w = (int)((off[s + 1] - o) >> 5);
  T acc = dzero<T>();
  const int32_t *cp = col + o + lane;
  const T *vp = val + o + lane;
#pragma unroll 8
  for (int e = 0; e < w; ++e) {
    const int32_t c = __ldg(cp + 32 * e);
    const T v = ld_nc(vp + 32 * e);
    if (c >= 0) acc += v * ((!HALO || c < n) ? ld_nc(x + c) : ld_nc(xh + (c - n)));
  }
  const int64_t row = s * 32 + lane;
  if (row < n) y[row] = mode ? b[row] - acc : acc;
}

// SELL-32 SpMV with more loads in flight: a warp takes SPW consecutive slices
// of width <= WM, issues all their column and value loads, then all x gathers
// (the gathers depend on the columns, so batching both levels is what hides
// the latency; one slice per warp left the kernel at 57 % of HBM).
// slist != nullptr: the warp's slices are slist[s0 + q] of a list of nslices
// entries (the interior / boundary slices of a distributed SpMV, whose halo
// exchange overlaps the interior part).
template <typename T, bool HALO, int SPW, int WM>
__global__ void __launch_bounds__(256) k_spmv_sell2(int64_t n, int64_t nslices, const int64_t *__restrict__ off,
                                                    const int32_t *__restrict__ col, const T *__restrict__ val,
                                                    const T *__restrict__ x, const T *__restrict__ xh, T *__restrict__ y,
                                                    int mode, const T *__restrict__ b, const int *__restrict__ done,
                                                    const int *__restrict__ slist = nullptr) {
  pdl_launch();
  pdl_wait();
  if (done && *done) return;
  const int64_t s0 = ((int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * SPW;
  if (s0 >= nslices) return;
  const int lane = threadIdx.x & 31;
  int c[SPW][WM];
  T v[SPW][WM];
  int64_t sid[SPW];
#pragma unroll
  for (int q = 0; q < SPW; ++q) sid[q] = s0 + q < nslices ? (slist ? (int64_t)slist[s0 + q] : s0 + q) : -1;
#pragma unroll
  for (int q = 0; q < SPW; ++q) {
    const int64_t s = sid[q];
    const int64_t o = s >= 0 ? off[s] : 0;
    const int w = s >= 0 ? (int)((off[s + 1] - o) >> 5) : 0;
#pragma unroll
    for (int e = 0; e < WM; ++e) {
      c[q][e] = e < w ? __ldg(col + o + 32 * e + lane) : -1;
      v[q][e] = e < w ? ld_nc(val + o + 32 * e + lane) : dzero<T>();
    }
  }
  T xv[SPW][WM];
#pragma unroll
  for (int q = 0; q < SPW; ++q)
#pragma unroll
    for (int e = 0; e < WM; ++e) {
      const int cc = c[q][e];
      xv[q][e] = cc < 0 ? dzero<T>() : ((!HALO || cc < n) ? ld_nc(x + cc) : ld_nc(xh + (cc - n)));
    }
#pragma unroll
  for (int q = 0; q < SPW; ++q) {
    T acc = dzero<T>();
#pragma unroll
    for (int e = 0; e < WM; ++e) acc += v[q][e] * xv[q][e];
    const int64_t row = sid[q] * 32 + lane;
    if (sid[q] >= 0 && row < n) y[row] = mode ? b[row] - acc : acc;
  }
}

// Warp per row (CSR) for matrices whose rows are long or very uneven (north_star:
// "warp-per-row or row-block variants picked by nnz/row"): lanes stride over a
// row's entries (coalesced column / value loads), a warp sum gives y_i.  SELL-32
// (one row per lane) would pad every lane of a slice to its longest row.
template <typename T, bool HALO>
__global__ void __launch_bounds__(256) k_spmv_wpr(int64_t n, const int64_t *__restrict__ ptr, const int32_t *__restrict__ col,
                                                  const T *__restrict__ val, const T *__restrict__ x,
                                                  const T *__restrict__ xh, T *__restrict__ y, int mode,
                                                  const T *__restrict__ b, const int *__restrict__ done) {
  pdl_launch();
  pdl_wait();
  if (done && *done) return;
  const int lane = threadIdx.x & 31;
  const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t row = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); row < n; row += nw) {
    T acc = dzero<T>();
    const int64_t p1 = ptr[row + 1];
    for (int64_t p = ptr[row] + lane; p < p1; p += 32) {
      const int32_t c = __ldg(col + p);
      acc += ld_nc(val + p) * ((!HALO || c < n) ? ld_nc(x + c) : ld_nc(xh + (c - n)));
    }
    acc = warp_sum(acc);
    if (lane == 0) y[row] = mode ? b[row] - acc : acc;
  }
}

// Several right-hand sides (NEXT-4): Y[:, c] = A X[:, c] for c < nr (column-major,
// leading dimension ld).  A warp loads the columns and values of its SELL slice
// once and gathers x for every right-hand side, so A is read once for all nr.
template <typename T, int WM>
__global__ void __launch_bounds__(256) k_spmv_multi(int64_t n, int64_t nslices, const int64_t *__restrict__ off,
                                                    const int32_t *__restrict__ col, const T *__restrict__ val,
                                                    const T *__restrict__ X, T *__restrict__ Y, int64_t ld, int nr) {
  const int64_t s = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (s >= nslices) return;
  const int lane = threadIdx.x & 31;
  const int64_t o = off[s];
  const int w = (int)((off[s + 1] - o) >> 5);
  int c[WM];
  T v[WM];
#pragma unroll
  for (int e = 0; e < WM; ++e) {
    c[e] = e < w ? __ldg(col + o + 32 * e + lane) : -1;
    v[e] = e < w ? ld_nc(val + o + 32 * e + lane) : dzero<T>();
  }
  const int64_t row = s * 32 + lane;
  for (int q = 0; q < nr; ++q) {
    const T *x = X + (size_t)q * ld;
    T acc = dzero<T>();
#pragma unroll
    for (int e = 0; e < WM; ++e)
      if (c[e] >= 0) acc += v[e] * ld_nc(x + c[e]);
    if (row < n) Y[(size_t)q * ld + row] = acc;
  }
}

// halo send buffer: buf[i] = src[idx[i]]
template <typename T>
__global__ void k_gather_idx(int64_t n, const int *__restrict__ idx, const T *__restrict__ src, T *__restrict__ buf,
                             const int *__restrict__ done) {
  if (done && *done) return;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    buf[i] = src[idx[i]];
}
// replicated last separator: dst[idx[i]] = src[i] (scatter) / dst[i] = src[idx[i]] (gather)
template <typename T>
__global__ void k_scatter_idx(int64_t n, const int *__restrict__ idx, const T *__restrict__ src, T *__restrict__ dst,
                              const int *__restrict__ done) {
  if (done && *done) return;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    dst[idx[i]] = src[i];
}

// ----------------------------------------------------------------- K4/K5/K9 trisolve
template <typename T>
struct TriDev {
  const int32_t *blk_lev;
  const int32_t *lev_slice;
  const int64_t *slice_off;
  const int32_t *slice_row;
  const int32_t *col;
  const T *val;
  const T *diag;
};

enum { TRI_DOWN = 0, TRI_UP = 1 };

// One CTA (CLUSTER=false) or one cluster of CPS CTAs (CLUSTER=true) per block.
// DOWN:  x[rows] = U^-1 L^-1 rhs[rows]                      (z1 of Alg. 2 l.2; C_last)
// UP:    t = F_l y_J (rows of the block) ; t = U^-1 L^-1 t ; x[rows] -= t   (Alg. 2 l.9)
// Every level of a sweep ends with a CTA / cluster barrier; rows of one level
// are independent and one warp handles one SELL slice (one row per lane).
template <typename T, bool CLUSTER>
__global__ void __launch_bounds__(256) k_trisolve(TriDev<T> Lp, TriDev<T> Up, const int64_t *__restrict__ blk, int mode,
                                                  const T *rhs, T *x, T *tmp, const int64_t *__restrict__ Fptr,
                                                  const int32_t *__restrict__ Fcol, const T *__restrict__ Fval,
                                                  int64_t Fbase, const int *__restrict__ done) {
  if (done && *done) return;
  int nct = 1, rank = 0;
  if (CLUSTER) {
    unsigned n;
    asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(n));
    nct = (int)n;
    rank = (int)cluster_ctarank();
  }
  const int b = blockIdx.x / nct;
  const int wpc = blockDim.x >> 5;
  const int gw = rank * wpc + (threadIdx.x >> 5);
  const int nw = nct * wpc;
  const int lane = threadIdx.x & 31;
  const int64_t r0 = blk[b], r1 = blk[b + 1];
  const int gt = rank * blockDim.x + threadIdx.x, nt = nct * blockDim.x;
  auto barrier = [&]() {
    if (CLUSTER) cluster_sync_all(); else __syncthreads();
  };
  auto ldv = [&](const T *p) -> T { return CLUSTER ? ld_cg(p) : *p; };
  const T *in;
  T *out;
  if (mode == TRI_DOWN) {
    in = rhs;
    out = x;
  } else {
    if (Fptr) {                                                 // t = F_l y_J (else precomputed in tmp)
      for (int64_t i = r0 + gt; i < r1; i += nt) {
        const int64_t li = i - Fbase;
        T acc = dzero<T>();
        for (int64_t p = Fptr[li]; p < Fptr[li + 1]; ++p) acc += Fval[p] * x[Fcol[p]];
        tmp[i] = acc;
      }
    }
    barrier();
    in = tmp;
    out = tmp;
  }
  // forward sweep, unit-lower L
  for (int v = Lp.blk_lev[b]; v < Lp.blk_lev[b + 1]; ++v) {
    for (int s = Lp.lev_slice[v] + gw; s < Lp.lev_slice[v + 1]; s += nw) {
      const int32_t row = Lp.slice_row[(int64_t)s * 32 + lane];
      const int64_t o = Lp.slice_off[s];
      const int w = (int)((Lp.slice_off[s + 1] - o) >> 5);
      if (row >= 0) {
        T acc = ldv(in + row);
        for (int e = 0; e < w; ++e) {
          const int32_t c = Lp.col[o + 32 * e + lane];
          if (c >= 0) acc -= Lp.val[o + 32 * e + lane] * ldv(out + c);
        }
        out[row] = acc;
      }
    }
    barrier();
  }
  // backward sweep, U with its diagonal
  for (int v = Up.blk_lev[b]; v < Up.blk_lev[b + 1]; ++v) {
    for (int s = Up.lev_slice[v] + gw; s < Up.lev_slice[v + 1]; s += nw) {
      const int32_t row = Up.slice_row[(int64_t)s * 32 + lane];
      const int64_t o = Up.slice_off[s];
      const int w = (int)((Up.slice_off[s + 1] - o) >> 5);
      if (row >= 0) {
        T acc = ldv(out + row);
        for (int e = 0; e < w; ++e) {
          const int32_t c = Up.col[o + 32 * e + lane];
          if (c >= 0) acc -= Up.val[o + 32 * e + lane] * ldv(out + c);
        }
        out[row] = acc / Up.diag[(int64_t)s * 32 + lane];
      }
    }
    barrier();
  }
  if (mode == TRI_UP)
    for (int64_t i = r0 + gt; i < r1; i += nt) x[i] = x[i] - ldv(tmp + i);   // y1 = z1 - U^-1 L^-1 F y2
}

// ----------------------------------------------------------------- K4/K5/K9 pipelined
// One CTA per block.  The factor data of the block's two sweeps is streamed
// chunk by chunk (<= 8 slices of one level) by 1D bulk copies (TMA,
// cp.async.bulk -> UBLKCP) into a pipe_stages<T>()-deep shared-memory ring
// with mbarrier completion, issued that many chunks ahead of the consumers; the
// solution values of the last `ring` packed positions stay in shared memory
// so a dependency costs a shared-memory load instead of an L2 round trip.
// One __syncthreads per chunk orders the levels and frees the stage.
struct ChunkDev {          // = ChunkDesc: blob offset / 128, blob bytes, first slice, ns << 1 | U flag
  int blob128, bytes, slice, nsflags;
};
template <typename T>
struct PipeDev {
  const unsigned char *blob;
  const ChunkDev *chunks;
  const int *blk_chunk;
  const int *blk_nl;
  const int *lpos;       // per stage row: packed L right-hand-side index
  long long row0;        // first row of the stage
  T *rhsL, *rhsU;        // packed right-hand sides of the L and U sweeps
  int ring;
};

__device__ inline unsigned smem_u32(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ inline void mbar_init(unsigned long long *b, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ inline void mbar_expect_tx(unsigned long long *b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ inline void bulk_g2s(void *dst, const void *src, unsigned bytes, unsigned long long *b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(b))
               : "memory");
}
__device__ inline void mbar_wait(unsigned long long *b, unsigned parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "LAB_WAIT:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@P1 bra DONE;\n\t"
      "bra LAB_WAIT;\n"
      "DONE:\n\t}" ::"r"(smem_u32(b)),
      "r"(parity)
      : "memory");
}

__device__ inline void mbar_arrive(unsigned long long *b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ inline bool mbar_test(unsigned long long *b, unsigned parity) {
  unsigned r;
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "mbarrier.test_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, P1;\n\t}"
      : "=r"(r)
      : "r"(smem_u32(b)), "r"(parity)
      : "memory");
  return r != 0;
}
__device__ inline void consumer_sync() { asm volatile("bar.sync 1, %0;" ::"r"(32 * PIPE_NW_DEV) : "memory"); }

__device__ inline void cp_async_8(void *dst, const void *src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ inline void cp_async_16(void *dst, const void *src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ inline void cp_async_arrive_noinc(unsigned long long *b) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(b)) : "memory");
}

template <typename T> __host__ __device__ constexpr int pipe_stages() { return sizeof(T) == 8 ? 3 : 2; }
template <typename T> __host__ __device__ constexpr size_t pipe_smem_bytes(int ring) {
  return (size_t)ring * sizeof(T) + (size_t)pipe_stages<T>() * (PIPE_SB_DEV + 32 * PIPE_NW_DEV * sizeof(T)) +
         (size_t)(2 * pipe_stages<T>() + 2) * 8;
}
__device__ inline void fence_proxy_async_global() { asm volatile("fence.proxy.async.global;" ::: "memory"); }

// Warp-specialised: warps 0..PIPE_NW-1 consume (one SELL slice of the chunk
// each); warp PIPE_NW produces.  Per stage s:
//   full[s]  the chunk's blob AND its packed right-hand sides landed (two bulk
//            copies, one complete_tx barrier);
//   empty[s] every consumer warp is done with stage s.
// The right-hand sides are packed in chunk order: the L sweep's by k_pack_rhs
// (a full-GPU kernel launched just before), the U sweep's (= the L results)
// by the consumers as they compute them (gate[1] after the last L chunk,
// crossed with fence.proxy.async so the bulk copies (async proxy) see the
// generic-proxy stores).  Consumers order the levels with a named
// barrier among themselves only.
template <typename T, bool FAR>
__global__ void __launch_bounds__(32 * (PIPE_NW_DEV + 1), 1) k_tri_pipe(PipeDev<T> P, const int64_t *__restrict__ blk, int mode,
                                                                     const T *rhs, T *x, T *tmp,
                                                                     const int64_t *__restrict__ Fptr,
                                                                     const int32_t *__restrict__ Fcol,
                                                                     const T *__restrict__ Fval, int64_t Fbase,
                                                                     const int *__restrict__ done, long long *dbg) {
  if (done && *done) return;
  constexpr int NS = pipe_stages<T>();
  constexpr int NCONS = 32 * PIPE_NW_DEV;
  extern __shared__ __align__(128) unsigned char smem[];
  const int R = P.ring;
  T *ring = reinterpret_cast<T *>(smem);
  unsigned char *stages = smem + (size_t)R * sizeof(T);
  T *rslot = reinterpret_cast<T *>(stages + (size_t)NS * PIPE_SB_DEV);
  unsigned long long *full = reinterpret_cast<unsigned long long *>(rslot + (size_t)NS * NCONS);
  unsigned long long *empty = full + NS;
  unsigned long long *gate = empty + NS;
  const int b = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int c0 = P.blk_chunk[b], nc = P.blk_chunk[b + 1] - c0;
  const int64_t r0 = blk[b], r1 = blk[b + 1];
  if (tid == 0) {
    for (int i = 0; i < NS; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], PIPE_NW_DEV);
    }
    mbar_init(&gate[1], PIPE_NW_DEV);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  // padding entries (value 0, column -1) read ring slot R-1; make it finite before
  // any position lands there (every other slot is written before it is read)
  if (tid == 0) ring[R - 1] = dzero<T>();
  __syncthreads();
  T *out = (mode == TRI_DOWN) ? x : tmp;
  if (warp == PIPE_NW_DEV) {                                       // ---- producer (one lane)
    if (lane != 0) return;
    bool g1 = false;
    // 16-byte descriptors, prefetched 4 chunks ahead in registers
    const int4 *dsc = reinterpret_cast<const int4 *>(P.chunks) + c0;
    int4 q0 = nc > 0 ? dsc[0] : make_int4(0, 0, 0, 0), q1 = nc > 1 ? dsc[1] : q0, q2 = nc > 2 ? dsc[2] : q0,
         q3 = nc > 3 ? dsc[3] : q0;
    for (int k = 0; k < nc; ++k) {
      const int4 d = q0;
      q0 = q1;
      q1 = q2;
      q2 = q3;
      if (k + 4 < nc) q3 = dsc[k + 4];
      const int st = k % NS;
      const int ns = d.w >> 1;
      const bool upper = d.w & 1;
      if (upper && !g1) { mbar_wait(&gate[1], 0); g1 = true; }
      if (k >= NS) mbar_wait(&empty[st], (unsigned)(((k / NS) - 1) & 1));
      const unsigned rb = (unsigned)(ns * 32 * sizeof(T));
      mbar_expect_tx(&full[st], (unsigned)d.y + rb);
      bulk_g2s(stages + (size_t)st * PIPE_SB_DEV, P.blob + (size_t)(unsigned)d.x * 128, (unsigned)d.y, &full[st]);
      bulk_g2s(rslot + (size_t)st * NCONS, (upper ? P.rhsU : P.rhsL) + (size_t)(unsigned)d.z * 32, rb, &full[st]);
      if (dbg && b == 0 && k < 4096) dbg[4 * k + 3] = clock64();
    }
    return;
  }
  // ---- consumer warps (the L right-hand sides were packed by k_pack_rhs)
  // The static per-chunk values of this lane (row, slice offsets, diagonal,
  // right-hand side) are fetched for chunk k+1 while chunk k is finishing, so
  // after the level barrier only the column/value and solution loads remain.
  struct Pre {
    const int *cp;
    const T *vp;
    T rhs, dg;
    int row, w, auxv, s0, flags, ok;
  };
  auto fetch = [&](int kk, Pre &p) {
    const int st = kk % NS;
    const int *hdr = reinterpret_cast<const int *>(stages + (size_t)st * PIPE_SB_DEV);
    const int4 h4 = *reinterpret_cast<const int4 *>(hdr);       // ns, s0, ne, flags
    const int ns = h4.x, ne = h4.z;
    const int H = (ns + 5 + 3) & ~3;
    const int *rows = hdr + H;
    const int *aux = rows + ns * 32;
    const T *diag = reinterpret_cast<const T *>(aux + ns * 32);
    const int *col = reinterpret_cast<const int *>(diag + ns * 32);
    const T *val = reinterpret_cast<const T *>(col + ne);
    p.s0 = h4.y;
    p.flags = h4.w;
    p.ok = 1;
    p.row = -1;
    if (warp < ns) {
      p.row = rows[warp * 32 + lane];
      const int e0 = hdr[4 + warp];
      p.w = (hdr[5 + warp] - e0) >> 5;
      p.cp = col + e0 + lane;
      p.vp = val + e0 + lane;
      p.rhs = rslot[(size_t)st * NCONS + warp * 32 + lane];
      p.dg = diag[warp * 32 + lane];
      p.auxv = aux[warp * 32 + lane];
    }
  };
  const int nL = P.blk_nl[b];
  Pre cur;
  cur.ok = 0;
  for (int k = 0; k < nc; ++k) {
    const int st = k % NS;
    if (dbg && b == 0 && tid == 0 && k < 4096) dbg[4 * k] = clock64();
    if (!cur.ok) {
      mbar_wait(&full[st], (unsigned)((k / NS) & 1));
      fetch(k, cur);
    }
    if (dbg && b == 0 && tid == 0 && k < 4096) dbg[4 * k + 1] = clock64();
    if (dbg && b == 0 && tid == 0 && k < 4096 && cur.row >= 0) {   // after the first column load
      const int c0 = cur.cp[0];
      dbg[5 * 4096 + k] = clock64() + (c0 == -7 ? 1 : 0);
    }
    const bool upper = cur.flags & 1;
    if (cur.row >= 0) {
      T acc = cur.rhs;
      const int w = cur.w;
      const int *cp = cur.cp;
      const T *vp = cur.vp;
      if (FAR) {
        // as below, with the rare "far" dependencies (c <= -2) read from global memory
        auto gx = [&](int c) -> T { return c >= 0 ? ring[c & (R - 1)] : (c <= -2 ? out[-c - 2] : dzero<T>()); };
        T a1 = dzero<T>(), a2 = dzero<T>(), a3 = dzero<T>();
        int e = 0;
#pragma unroll 2
        for (; e + 4 <= w; e += 4) {
          const int c0 = cp[32 * e], c1 = cp[32 * (e + 1)], c2 = cp[32 * (e + 2)], c3 = cp[32 * (e + 3)];
          const T v0 = vp[32 * e], v1 = vp[32 * (e + 1)], v2 = vp[32 * (e + 2)], v3 = vp[32 * (e + 3)];
          acc -= v0 * gx(c0);
          a1 -= v1 * gx(c1);
          a2 -= v2 * gx(c2);
          a3 -= v3 * gx(c3);
        }
        if (e < w) a1 -= vp[32 * e] * gx(cp[32 * e]);
        if (e + 1 < w) a2 -= vp[32 * (e + 1)] * gx(cp[32 * (e + 1)]);
        if (e + 2 < w) a3 -= vp[32 * (e + 2)] * gx(cp[32 * (e + 2)]);
        acc = (acc + a1) + (a2 + a3);
      } else {
        // branch-free: padding has value 0 and column -1 (ring slot R-1, finite
        // because the ring is zero-initialised); two partial sums shorten the
        // dependent DFMA chain
        // four partial sums: the dependent DFMA chain of a ~10-entry row is 3 deep
        T a1 = dzero<T>(), a2 = dzero<T>(), a3 = dzero<T>();
        int e = 0;
#pragma unroll 2
        for (; e + 4 <= w; e += 4) {
          const int c0 = cp[32 * e], c1 = cp[32 * (e + 1)], c2 = cp[32 * (e + 2)], c3 = cp[32 * (e + 3)];
          const T v0 = vp[32 * e], v1 = vp[32 * (e + 1)], v2 = vp[32 * (e + 2)], v3 = vp[32 * (e + 3)];
          acc -= v0 * ring[c0 & (R - 1)];
          a1 -= v1 * ring[c1 & (R - 1)];
          a2 -= v2 * ring[c2 & (R - 1)];
          a3 -= v3 * ring[c3 & (R - 1)];
        }
        if (e < w) a1 -= vp[32 * e] * ring[cp[32 * e] & (R - 1)];
        if (e + 1 < w) a2 -= vp[32 * (e + 1)] * ring[cp[32 * (e + 1)] & (R - 1)];
        if (e + 2 < w) a3 -= vp[32 * (e + 2)] * ring[cp[32 * (e + 2)] & (R - 1)];
        acc = (acc + a1) + (a2 + a3);
      }
      if (dbg && b == 0 && tid == 0 && k < 4096) {
        const double probe = dabs2(acc);
        dbg[4 * 4096 + k] = clock64() + (probe != probe ? 1 : 0);
      }
      if (upper) acc = acc * cur.dg;                              // diag holds 1 / u_ii
      else P.rhsU[cur.auxv] = acc;                                 // right-hand side of the U sweep
      ring[((cur.s0 + warp) * 32 + lane) & (R - 1)] = acc;
      out[cur.row] = acc;
    }
    const bool level_end = cur.flags & 2;
    __syncwarp();
    if (dbg && b == 0 && tid == 0 && k < 4096) dbg[4 * k + 2] = clock64();
    if (lane == 0) mbar_arrive(&empty[st]);
    cur.ok = 0;
    if (k + 1 < nc) {
      const int st1 = (k + 1) % NS;
      if (mbar_test(&full[st1], (unsigned)(((k + 1) / NS) & 1))) fetch(k + 1, cur);
    }
    if (k == nL - 1) {                                             // L sweep done: release the U right-hand sides
      fence_proxy_async_global();
      __threadfence();
      __syncwarp();
      if (lane == 0) mbar_arrive(&gate[1]);
    }
    if (level_end) consumer_sync();                                // rows of one level are independent
  }
  if (mode == TRI_UP)
    for (int64_t i = r0 + tid; i < r1; i += NCONS) x[i] = x[i] - tmp[i];   // y1 = z1 - U^-1 L^-1 F y2
}

// sum_p val[p] * g(col[p]) over p in [p0, p1) in p order (the plain loop's rounding);
// the column/value loads of 8 entries, then their 8 gathers, are issued together, so
// a short row costs two dependent round trips instead of two per entry.
template <typename T, typename Gather>
__device__ inline T csr_dot(int64_t p0, int64_t p1, const int32_t *__restrict__ col, const T *__restrict__ val,
                            Gather g) {
  T acc = dzero<T>();
  for (int64_t q = p0; q < p1; q += 8) {
    int64_t c[8];
    T v[8], x[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const bool ok = q + u < p1;
      c[u] = ok ? (int64_t)col[q + u] : -1;
      v[u] = ok ? val[q + u] : dzero<T>();
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) x[u] = c[u] >= 0 ? g(c[u]) : dzero<T>();
#pragma unroll
    for (int u = 0; u < 8; ++u)
      if (q + u < p1) acc += v[u] * x[u];
  }
  return acc;
}

// ----------------------------------------------------------------- K4/K5/K9 register-prefetched
// One CTA per block, NW warps.  The slices of a
// sweep (level order) go round-robin to the consumer warps: slice s -> warp
// s mod NW, so a warp's next slice is NW slices on and its record (values,
// 16-bit ring slots, output position, 1/u_ii) is loaded straight into registers
// right after the warp's current slice — no shared-memory staging of the factor
// stream, whose 128 B/clk port was the floor of k_tri_pipe.  Levels are
// separated by named barriers among the consumer warps; a dependency is a
// shared-memory load from the ring of the last `ring` solution values (the
// setup proves every dependency is still in the window, RegPack::far == 0).
// (An L2-prefetch helper warp, paced by a level counter, was measured: no gain
// on level 0 and 1.8x slower levels 1/2 of C5 while it polls; removed.)
// NB record buffers per warp (see the slice loop): 2 with NW = 15, or 1 with
// the wide NW = 23 variant, whose register budget is 88.
// DOWN: x[rows] = U^-1 L^-1 rhs (rhsL = rhs packed in L order by k_pack_rhs)
// UP:   x[rows] -= U^-1 L^-1 (F_l y_J) (rhsL = F_l y_J packed by k_pack_rhs)
// The L results go to `mid` at their packed U position: the U sweep's right-hand
// sides, read after the sweep-transition barrier.
template <typename T>
struct RegDev {
  const unsigned char *data;   // fixed-size records (RegPack)
  const unsigned short *slev;  // level of every record in its sweep
  long long rec_bytes;
  const int *binfo;
  const int *lev_off;
  const T *rhsL;
  T *mid;
  const T *xU;             // UP, one column: the level's x in U-packed order (k_pack_f); else null (tmp path)
  T *xP;                   // DOWN, one column: write the result in U-packed order here instead of x[row]
  int ring;
  long long *dbg;          // debug trace (block 0): 8 words per slice, 2048 slices per sweep
  int max_slices;          // L + U records of the largest block (shared-memory level table)
  // several right-hand sides (NEXT-4): column blockIdx.y works on x/tmp + col*ldx
  // and rhsL/mid + col*rs (0 for one column); the factor records are shared
  long long ldx, rsL, rsU;
  // split form (plan.hpp RegPack, Q > 1): a Q-CTA cluster per block
  int Q;
  int imp_L, imp_U;            // import areas after the ring (entries)
  int plev_L, plev_U;          // counter / expectation table sizes
  const unsigned short *sneed; // per record: producer level needed + 1 (0 none)
  const unsigned short *xexp;  // expected exporting slices per producer level
  int xp;                      // one-CTA imports (RegPack::xmode): records carry exp[32]
  // tail form (TAIL, plan.hpp TailPack): three sweeps, each with its right-hand side
  // ra[pos + roff] (- rb[pos + roff]), pos = stage slice * 32 + lane, and its store:
  // stm 0: st[out] (L sweeps: Ucat position; U sweeps: the row), 1: st[pos + roff]
  const T *ra[3];
  const T *rb[3];
  T *st[3];
  long long roff[3];
  int upper[3];
  int stm[3];
};
#ifdef GEMSLR_TRACE
constexpr bool kRegTrace = true;         // clock64 trace of block 0 (tools/trace_reg.py; build with GEMSLR_TRACE=1)
#else
constexpr bool kRegTrace = false;
#endif
__host__ __device__ constexpr size_t al16(size_t b) { return (b + 15) & ~(size_t)15; }
// [ring | imports] T, 16 bytes, [mbarriers u64 | expectations u16] (split), level
// table u16, [need table u16] (split)
template <typename T> __host__ __device__ inline size_t reg_smem_bytes(int ring, int max_slices, int imp = 0, int plev = 0,
                                                                       bool split = false) {
  return (size_t)(ring + imp) * sizeof(T) + 16 + (split ? al16((size_t)plev * 8) + al16((size_t)plev * 2) : 0) +
         al16((size_t)max_slices * 2) * (split ? 2 : 1);
}
constexpr int REG_BINFO = 16;            // ints per block in RegDev::binfo (= REG_BINFO_INTS)
constexpr int REG_LA_DEV = 3;            // = REG_LA (look-ahead new columns)
constexpr int REG_LEV_MASK = 0xffff;

// DSMEM hand-off of the split form: every exported value is an asynchronous
// remote store (st.async) that completes its bytes on the consumer's mbarrier of
// the producer's level; the consumer set each barrier's expected bytes at start and
// waits on it (local try_wait) only when a slice reads that level's values.  No
// fence on either side: the producer never stalls on its stores.
__device__ inline unsigned mapa_shared(unsigned addr, unsigned rank) {
  unsigned r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}
__device__ inline void st_async_cluster(unsigned addr, double v, unsigned mbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.f64 [%0], %1, [%2];" ::"r"(addr), "d"(v), "r"(mbar)
               : "memory");
}
__device__ inline void st_async_cluster(unsigned addr, cd v, unsigned mbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];" ::"r"(addr),
               "d"(v.x), "d"(v.y), "r"(mbar)
               : "memory");
}

// Level v of a sweep ends at named barrier 1 + v % 15 (15 ids in rotation).
// A warp that computes in level v + 1 SYNCS there (arrive + wait); every other
// warp only ARRIVES (bar.arrive, no wait) — right after its slice, before its
// global stores and record loads, so those overlap the following levels.  A
// warp may arrive at level v only once instance v - 15 of the id is complete:
// with NW <= 15 that always holds (a warp runs at most NW - 1 levels ahead);
// wider variants sync instead of arriving when they would get further ahead.
template <int NW> __device__ inline void reg_arrive(int v) {
  asm volatile("bar.arrive %0, %1;" ::"r"(1 + v % 15), "n"(32 * NW) : "memory");
}
template <int NW> __device__ inline void reg_sync(int v) {
  asm volatile("bar.sync %0, %1;" ::"r"(1 + v % 15), "n"(32 * NW) : "memory");
}
template <int NW> __device__ inline void reg_arrive_id(int id) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "n"(32 * NW) : "memory");
}
template <int NW> __device__ inline void reg_sync_id(int id) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "n"(32 * NW) : "memory");
}
template <int NW> __device__ inline void reg_sync_all() { asm volatile("bar.sync 0, %0;" ::"n"(32 * NW) : "memory"); }

// 16 bytes of values per lane and load: VE entries (2 doubles / 1 complex)
template <typename T> struct Vec16;
template <> struct Vec16<double> { using type = double2; static constexpr int VE = 2; };
template <> struct Vec16<cd> { using type = double2; static constexpr int VE = 1; };
template <typename T> __device__ inline T vec_get(const double2 &u, int k);
template <> __device__ inline double vec_get<double>(const double2 &u, int k) { return k ? u.y : u.x; }
template <> __device__ inline cd vec_get<cd>(const double2 &u, int) { return cd{u.x, u.y}; }

template <typename T, int W>
struct RegBuf {
  static constexpr int VE = Vec16<T>::VE;
  static constexpr int NV = (W + VE - 1) / VE;   // 16-byte value loads
  static constexpr int W8 = (W + 7) / 8;         // 16-byte slot loads (8 x uint16)
  double2 v[NV];
  uint4 c[W8];
  T rhs, dg, xo;
  int out;
  int exp;                                       // split: import index at the consumer (-1 none)
  __device__ T val(int e) const { return vec_get<T>(v[e / VE], e % VE); }
  __device__ unsigned slot(int e) const {
    const uint4 &q = c[e / 8];
    const int k = (e % 8) / 2;
    const unsigned w = k == 0 ? q.x : k == 1 ? q.y : k == 2 ? q.z : q.w;
    return (e & 1) ? (w >> 16) : (w & 0xffffu);
  }
};

#ifndef SPLIT_EXPORT_FIRST
#define SPLIT_EXPORT_FIRST 0
#endif
template <typename T, int W, int NW, int NB, bool SPLIT = false, int LA = 0, bool TAIL = false>
__global__ void __launch_bounds__(32 * (NW + (SPLIT ? 1 : 0)), 1) k_tri_reg(RegDev<T> P, int mode, T *x, T *tmp,
                                                            const int *__restrict__ done) {
  pdl_launch();
  // An iteration queued after convergence exits before its prologue.  (The flag only
  // goes 0 -> 1 within a cycle, so reading it before griddepcontrol.wait is safe: a
  // stale 0 falls through to the check after the wait.)  Not in the split form: the
  // CTAs of a cluster must take the same decision (they meet at cluster barriers).
  if (!SPLIT && done && *(volatile const int *)done) return;
  if (blockIdx.y) {                                                // right-hand side column blockIdx.y (NEXT-4)
    x += (size_t)blockIdx.y * P.ldx;
    tmp += (size_t)blockIdx.y * P.ldx;
    P.rhsL += (size_t)blockIdx.y * P.rsL;
    P.mid += (size_t)blockIdx.y * P.rsU;
  }
  extern __shared__ __align__(128) unsigned char smem[];
  T *ring = reinterpret_cast<T *>(smem);
  const int R = P.ring;
  const int IL = SPLIT ? P.imp_L : 0, PL = SPLIT ? P.plev_L : 0, PLU = SPLIT ? P.plev_L + P.plev_U : 0;
  unsigned char *tail = smem + (size_t)(R + P.imp_L + P.imp_U) * sizeof(T) + 16;   // (imports: 0 unless split / xp)
  // split: the import warp's progress, per sweep: producer levels whose values landed
  volatile int *ready = reinterpret_cast<volatile int *>(tail - 16);
  unsigned long long *mb = reinterpret_cast<unsigned long long *>(tail);       // split: one mbarrier per producer level
  unsigned short *xex = reinterpret_cast<unsigned short *>(tail + al16((size_t)PLU * 8));
  unsigned short *lvt = reinterpret_cast<unsigned short *>(SPLIT ? tail + al16((size_t)PLU * 8) + al16((size_t)PLU * 2) : tail);
  unsigned short *ndt = lvt + al16((size_t)P.max_slices * 2) / 2;             // split: producer level needed + 1
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // The block's info goes through shared memory: a register loaded from global
  // memory shares a scoreboard slot with the prefetch loads issued later, and
  // every later read of it would wait for those (shared loads use another slot).
  __shared__ int bis[REG_BINFO];
  if (tid < REG_BINFO) bis[tid] = P.binfo[REG_BINFO * blockIdx.x + tid];
  __syncthreads();
  const int *bi = bis;
  {                                                                // level table of the block's records (L then U)
    const int f = bi[0], nl = bi[1] + bi[4] + (TAIL ? bi[7] : 0);  // U records follow the L records of the block
    constexpr int U = 8;                                           // independent loads in flight per thread
    const int nt = blockDim.x;
    int i = tid;
    for (; i + (U - 1) * nt < nl; i += U * nt) {
      unsigned short v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) v[u] = P.slev[f + i + u * nt];
#pragma unroll
      for (int u = 0; u < U; ++u) lvt[i + u * nt] = v[u];
    }
    for (; i < nl; i += nt) lvt[i] = P.slev[f + i];
    if constexpr (SPLIT) {
      for (int j = tid; j < nl; j += nt) ndt[j] = P.sneed[f + j];
      for (int j = tid; j < PLU; j += nt) {                        // producer level j: expected values
        const int in_l = j < PL;
        const int u = in_l ? j : j - PL;
        const unsigned e = in_l ? (u < bi[13] ? P.xexp[bi[12] + u] : 0u) : (u < bi[15] ? P.xexp[bi[14] + u] : 0u);
        xex[j] = (unsigned short)e;
        mbar_init(&mb[j], 1);
      }
    }
  }
  for (int i = tid; i < R; i += blockDim.x) ring[i] = dzero<T>();
  __syncthreads();
  // split: the neighbours' import areas and barriers (L exports go to q + 1, U to q - 1)
  unsigned rimp[2] = {0, 0}, rmb[2] = {0, 0};
  if constexpr (SPLIT) {
    if (tid == 0) asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncthreads();
    for (int j = tid; j < PLU; j += blockDim.x) {                 // arm: the phase completes when the bytes land
      const unsigned bytes = (unsigned)xex[j] * (unsigned)sizeof(T);
      if (bytes) mbar_expect_tx(&mb[j], bytes);
      else mbar_arrive(&mb[j]);
    }
    const unsigned q = cluster_ctarank();
    const unsigned rs = smem_u32(ring), ms = smem_u32(mb);
    if (q + 1 < (unsigned)P.Q) { rimp[0] = mapa_shared(rs + (unsigned)(R * sizeof(T)), q + 1); rmb[0] = mapa_shared(ms, q + 1); }
    if (q > 0) {
      rimp[1] = mapa_shared(rs + (unsigned)((R + IL) * sizeof(T)), q - 1);
      rmb[1] = mapa_shared(ms + (unsigned)(PL * 8), q - 1);
    }
    if (tid < 2) ready[tid] = -1;
    cluster_sync_all();                                            // barriers armed before any export
  }
  pdl_wait();                                                      // the prologue above reads setup data only
  if (done && *done) return;
  if (SPLIT && warp == NW) {
    // the import warp: follows the producer levels' barriers in order (L, then U)
    // and publishes how far the imports have landed; the compute warps only read
    // that word (a barrier check costs ~150 cycles; walking them on the critical
    // path made every consumer level 2-3x slower)
    if constexpr (SPLIT) {
      for (int sw2 = 0; sw2 < 2; ++sw2) {
        const int np = sw2 ? bi[15] : bi[13], off = sw2 ? PL : 0;
        for (int u = 0; u < np; ++u) {
          if (xex[off + u])
            while (!mbar_test(&mb[off + u], 0)) __nanosleep(20);
          __syncwarp();
          if (lane == 0) {
            __threadfence_block();
            ready[sw2] = u;
          }
        }
      }
    }
  } else {
  const bool inplace = !TAIL && mode == TRI_UP && P.xU != nullptr;
  const size_t RB = (size_t)P.rec_bytes;
  using Buf = RegBuf<T, W>;
  constexpr int NV = Buf::NV, W8 = Buf::W8;
#pragma unroll 1
  for (int sw = 0; sw < (TAIL ? 3 : 2); ++sw) {
    const bool upper = TAIL ? P.upper[sw] != 0 : sw == 1;
    const int r0 = bi[3 * sw], ns = bi[3 * sw + 1], nlev = bi[3 * sw + 2], gbase = TAIL ? bi[9 + sw] : bi[10 + sw];
    const int lvbase = TAIL ? (sw == 0 ? 0 : sw == 1 ? bi[1] : bi[1] + bi[4]) : (upper ? bi[1] : 0);
    // tail form: this sweep's right-hand sides and store (uniform selects, no indexed parameter load)
    const T *t_ra = nullptr, *t_rb = nullptr;
    T *t_st = nullptr;
    long long t_off = 0;
    int t_stm = 0;
    if constexpr (TAIL) {
      t_ra = sw == 0 ? P.ra[0] : sw == 1 ? P.ra[1] : P.ra[2];
      t_rb = sw == 0 ? P.rb[0] : sw == 1 ? P.rb[1] : P.rb[2];
      t_st = sw == 0 ? P.st[0] : sw == 1 ? P.st[1] : P.st[2];
      t_off = sw == 0 ? P.roff[0] : sw == 1 ? P.roff[1] : P.roff[2];
      t_stm = sw == 0 ? P.stm[0] : sw == 1 ? P.stm[1] : P.stm[2];
    }
    // Issues the loads of slice s; every address is arithmetic on s, so the
    // warp never waits here and reaches the next barrier right after its slice.
    auto load = [&](Buf &B, int s) {
      if (s >= ns) return;
      const unsigned char *rec = P.data + (size_t)(r0 + s) * RB;
      const double2 *vp = reinterpret_cast<const double2 *>(rec) + lane;
      const uint4 *cp = reinterpret_cast<const uint4 *>(rec + (size_t)W * 32 * sizeof(T)) + lane;
      const int *op = reinterpret_cast<const int *>(rec + (size_t)W * 32 * sizeof(T) + (size_t)W8 * 512);   // out[]
#pragma unroll
      for (int k = 0; k < NV; ++k) B.v[k] = ld_na(vp + 32 * k);   // streamed once: no L1 allocation (-3 % on C5 level 0)
#pragma unroll
      for (int j = 0; j < W8; ++j) B.c[j] = ld_na(cp + 32 * j);
      B.out = __ldg(op + lane);
      if constexpr (SPLIT || TAIL) B.exp = __ldg(reinterpret_cast<const int *>(op + 32 + 32 * (int)(sizeof(T) / 4)) + lane);
      else B.exp = P.xp ? __ldg(reinterpret_cast<const int *>(op + 32 + 32 * (int)(sizeof(T) / 4)) + lane) : -1;
      const size_t ri = (size_t)(gbase + s) * 32 + lane;
      if constexpr (TAIL) {                                        // written by earlier kernels or sweeps: L2
        if (upper) B.dg = ld_nc(reinterpret_cast<const T *>(op + 32) + lane);
        B.rhs = ld_cg(t_ra + ri + t_off);
        // (subtracted at the solve: a use here would wait for every load just issued)
        B.xo = t_rb ? ld_cg(t_rb + ri + t_off) : dzero<T>();
        return;
      }
      if (upper) {
        B.dg = ld_nc(reinterpret_cast<const T *>(op + 32) + lane);
        B.rhs = ld_cg(P.mid + ri);                                 // written by this CTA's L sweep
        if (inplace) B.xo = ld_nc(P.xU + ri);
      } else {
        B.rhs = ld_nc(P.rhsL + ri);
      }
    };
    // Level barriers.  cur = the next level this warp has not yet arrived at;
    // known = the last level it saw complete.  Level v ends at named barrier
    // 1 + v % 15, so arriving at v needs instance v - 15 complete (known >= v - 15):
    // with NW <= 15 that always holds (a warp's next slice is NW slices on, so
    // it is at most NW - 1 levels ahead); with more warps a warp that would get
    // further ahead syncs instead of arriving.
    // cid = 1 + cur % 15, kept incrementally (no division on the critical path).
    int cur = 0, known = -1, cid = 1;
    auto pass = [&](bool may_block) {                              // arrive at level cur (no slice of this warp in it)
      if (NW > 15 && cur - known >= 15) {
        if (!may_block) return false;
        reg_sync_id<NW>(cid);
        known = cur;
      } else {
        reg_arrive_id<NW>(cid);
      }
      ++cur;
      cid = cid == 15 ? 1 : cid + 1;
      return true;
    };
    auto wait_level = [&](int lv) {                                // this warp computes in level lv next
      while (cur < lv - 1) pass(true);                             // levels with no slice of this warp
      if (cur < lv) {                                               // wait for level lv - 1 to complete
        reg_sync_id<NW>(cid);
        known = cur;
        ++cur;
        cid = cid == 15 ? 1 : cid + 1;
      }
    };
    // Look-ahead: the old group (columns [0, wo): levels before the previous one,
    // imports) is summed after the barrier two levels back, while the previous
    // level still runs; after the last barrier only the new group (the 1-3 entries
    // on the previous level) remains on the critical path.
    constexpr int WO = W - LA;                                     // old columns [0, WO), new [WO, W)
    auto solve_old = [&](const Buf &B) {
      T a0 = B.rhs, a1 = dzero<T>(), a2 = dzero<T>(), a3 = dzero<T>();
      if constexpr (TAIL) a1 = -B.xo;
#pragma unroll
      for (int e = 0; e < WO; e += 4) {
        a0 -= B.val(e) * ring[B.slot(e)];
        if (e + 1 < WO) a1 -= B.val(e + 1) * ring[B.slot(e + 1)];
        if (e + 2 < WO) a2 -= B.val(e + 2) * ring[B.slot(e + 2)];
        if (e + 3 < WO) a3 -= B.val(e + 3) * ring[B.slot(e + 3)];
      }
      return (a0 + a1) + (a2 + a3);
    };
    auto solve_new = [&](const Buf &B, T acc) {
      T b1 = dzero<T>();
#pragma unroll
      for (int e = WO; e < W; ++e) {
        if (((e - WO) & 1) == 0) acc -= B.val(e) * ring[B.slot(e)];
        else b1 -= B.val(e) * ring[B.slot(e)];
      }
      acc = acc + b1;
      if (upper) acc = acc * B.dg;
      return acc;
    };
    // x_i = (rhs_i - sum_j a_ij x_j) [/ u_ii]: W ring gathers, four partial sums
    auto solve = [&](const Buf &B, int s) {
      const bool tr = !SPLIT && kRegTrace && P.dbg && blockIdx.x == 0 && lane == 0 && s < 2048;
      long long *tp = tr ? P.dbg + 8 * (sw * 2048 + s) : nullptr;
      if (tr) { tp[2] = clock64(); tp[6] = lvt[lvbase + s] & REG_LEV_MASK; tp[7] = warp; tp[0] = tp[2]; }
      if (tr) {
        const double pr = dabs2(B.val(0)) + dabs2(B.val(W - 1)) + (double)B.slot(0) + (double)B.slot(W - 1) + dabs2(B.rhs);
        tp[4] = clock64() + (pr != pr ? 1 : 0);
        const double q = dabs2(ring[B.slot(0)]) + dabs2(ring[B.slot(W - 1)]);
        tp[5] = clock64() + (q != q ? 1 : 0);
      }
      T acc = B.rhs, a1 = dzero<T>(), a2 = dzero<T>(), a3 = dzero<T>();
      if constexpr (TAIL) a1 = -B.xo;
#pragma unroll
      for (int e = 0; e < W; e += 4) {
        acc -= B.val(e) * ring[B.slot(e)];
        if (e + 1 < W) a1 -= B.val(e + 1) * ring[B.slot(e + 1)];
        if (e + 2 < W) a2 -= B.val(e + 2) * ring[B.slot(e + 2)];
        if (e + 3 < W) a3 -= B.val(e + 3) * ring[B.slot(e + 3)];
      }
      acc = (acc + a1) + (a2 + a3);
      if (tr) { const double pr = dabs2(acc); tp[1] = clock64() + (pr != pr ? 1 : 0); tp[3] = tp[1]; }
      if (upper) acc = acc * B.dg;
      return acc;
    };
    auto publish = [&](const Buf &B, int s, const T &acc) {
      if (B.out >= 0) ring[(s * 32 + lane) & (R - 1)] = acc;
      if constexpr (!SPLIT) {                                      // imports: far / cross readers (xp, tail form)
        if (B.exp >= 0) ring[R + B.exp] = acc;
      }
    };
    // Done with the current level: arrive now at it and at every later level
    // before nxt, the level of this warp's next slice (bar.arrive does not wait),
    // so the stores and the record loads that follow never delay a level; the
    // level right before nx's is synced on when nx is computed.
    // (Look-ahead: the arrivals stop one level earlier — the level two before nxt is
    // synced on, so the next slice's old group may read it.)
    constexpr int DL = LA > 0 ? 2 : 1;
    auto depart = [&](int nxt) {
      if (cur < nxt - DL && pass(false)) {                         // the current level: straight-line arrival
#pragma unroll 1
        while (cur < nxt - DL && pass(false)) {}
      }
    };
    auto level_of = [&](int t) { return t < ns ? (int)(lvt[lvbase + t] & REG_LEV_MASK) : nlev; };
    // split: wait until the neighbour's exports this slice reads have landed (the
    // producer levels up to need - 1, monotone per warp); one acquire fence when any
    int rdy = -1;
    const unsigned rimp_sw = upper ? rimp[1] : rimp[0], rmb_sw = upper ? rmb[1] : rmb[0];
    // (test_wait polling: a try_wait suspends the warp and a remote st.async
    // completion did not wake it before the suspend limit — microseconds per wait)
    auto wait_imports = [&](int s_) {
      if constexpr (SPLIT) {
        const int needu = (int)ndt[lvbase + s_] - 1;
        if (rdy >= needu) return;
        while ((rdy = ready[sw]) < needu) {}
        __threadfence_block();                                     // acquire the landed values
      }
    };
    // split: this slice's exported values to the neighbour's import area, each
    // completing its bytes on the neighbour's barrier of this slice's level
    auto export_ = [&](const Buf &B, int s_, const T &acc) {
      if constexpr (SPLIT) {
        if (B.exp >= 0)
          st_async_cluster(rimp_sw + (unsigned)(B.exp * (int)sizeof(T)), acc,
                           rmb_sw + (unsigned)(lvt[lvbase + s_] & REG_LEV_MASK) * 8u);
      }
    };
    // The global stores are read only after the sweep-transition barrier.
    auto store = [&](const Buf &B, const T &acc, int s) {
      if constexpr (TAIL) {
        if (t_stm) t_st[(size_t)(gbase + s) * 32 + lane + t_off] = acc;
        else if (B.out >= 0) t_st[B.out] = acc;
        return;
      }
      if (upper && P.xP) {                                         // coalesced: U-packed position of the row
        P.xP[(size_t)(gbase + s) * 32 + lane] = acc;
        return;
      }
      if (B.out >= 0) {
        if (!upper) P.mid[B.out] = acc;
        else if (inplace) x[B.out] = B.xo - acc;                   // y1 = z1 - U^-1 L^-1 F y2 (Alg. 2 l.9)
        else if (mode == TRI_UP) tmp[B.out] = acc;                 // x -= tmp after the sweep
        else x[B.out] = acc;
      }
    };
    // The warp's slices are NW apart.  Its record loads are issued right after
    // a slice and waited for at the next: ptxas tracks every global load on one
    // scoreboard and the first read of a loaded register waits for all of them,
    // so the prefetch lead is about one slice period of the warp whatever the
    // buffering; more consumer warps lengthen it.  NB = 1: one buffer, refilled
    // with the next slice (the NW = 23 variant, 80 registers).  NB = 2: two
    // buffers alternating, refilled two slices ahead (NW = 15; measured best
    // for stages with 1-2 slices per level).
    // split trace (GEMSLR_TRACE=1, tools/trace_split.py): CTAs 0..Q-1 of block 0, lane 0
    // of every slice: clock64 before the level wait, after the import wait, after the
    // solve, and the slice's level; per CTA one (clock64, globaltimer) pair at start
    const bool str = SPLIT && kRegTrace && P.dbg && blockIdx.x < (unsigned)P.Q && lane == 0;
    long long *sbase = str ? P.dbg + 16 + (size_t)blockIdx.x * (2 * 2048 * 4) + (size_t)sw * 2048 * 4 : nullptr;
    if (str && sw == 0 && warp == 0) {
      long long g;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g));
      P.dbg[2 * blockIdx.x] = clock64();
      P.dbg[2 * blockIdx.x + 1] = g;
    }
    Buf A, B;
    int s = warp;
    load(A, s);
    if (NB == 2) load(B, s + NW);
#pragma unroll 1
    while (s < ns) {
      int nxt = level_of(s + NW);                                  // read before the barrier: off the critical path
      const long long tq0 = (str && s < 2048) ? clock64() : 0;
      const int lv = lvt[lvbase + s];
      T a0;
      if constexpr (LA > 0) {
        wait_level(lv - 1);                                        // the level two back is complete
        wait_imports(s);
        const T p0 = solve_old(A);
        wait_level(lv);                                            // the previous level is complete
        a0 = solve_new(A, p0);
      } else {
        wait_level(lv);
        wait_imports(s);
        a0 = solve(A, s);
      }
      const long long tq1 = (str && s < 2048) ? clock64() : 0;
      publish(A, s, a0);
      if (str && s < 2048) {
        const double pr = dabs2(a0);
        long long *q4 = sbase + 4 * s;
        q4[0] = tq0; q4[1] = tq1; q4[2] = clock64() + (pr != pr ? 1 : 0); q4[3] = (lvt[lvbase + s] & REG_LEV_MASK) | ((long long)ndt[lvbase + s] << 32);
      }
      if (SPLIT_EXPORT_FIRST) export_(A, s, a0);
      depart(nxt);
      if (!SPLIT_EXPORT_FIRST) export_(A, s, a0);
      store(A, a0, s);
      load(A, s + NB * NW);
      s += NW;
      if (NB == 2) {
        if (s >= ns) break;
        nxt = level_of(s + NW);
        const long long tr0 = (str && s < 2048) ? clock64() : 0;
        const int lv2 = lvt[lvbase + s];
        T a1;
        if constexpr (LA > 0) {
          wait_level(lv2 - 1);
          wait_imports(s);
          const T p1 = solve_old(B);
          wait_level(lv2);
          a1 = solve_new(B, p1);
        } else {
          wait_level(lv2);
          wait_imports(s);
          a1 = solve(B, s);
        }
        const long long tr1 = (str && s < 2048) ? clock64() : 0;
        publish(B, s, a1);
        if (str && s < 2048) {
          const double pr = dabs2(a1);
          long long *q4 = sbase + 4 * s;
          q4[0] = tr0; q4[1] = tr1; q4[2] = clock64() + (pr != pr ? 1 : 0); q4[3] = (lvt[lvbase + s] & REG_LEV_MASK) | ((long long)ndt[lvbase + s] << 32);
        }
        if (SPLIT_EXPORT_FIRST) export_(B, s, a1);
        depart(nxt);
        if (!SPLIT_EXPORT_FIRST) export_(B, s, a1);
        store(B, a1, s);
        load(B, s + 2 * NW);
        s += NW;
      }
    }
    while (cur < nlev) pass(true);
    __threadfence_block();
    reg_sync_all<NW>();                                            // sweep transition: mid / tmp visible, ring free
  }
  if (!TAIL && mode == TRI_UP && !inplace) {                       // y1 = z1 - U^-1 L^-1 F y2 (Alg. 2 l.9)
    constexpr int U = 8;                                           // 8 independent rows in flight per thread
    const int i0 = bi[8], i1 = bi[9];
    int i = i0 + tid;
    for (; i + (U - 1) * 32 * NW < i1; i += U * 32 * NW) {
      T a[U], t[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        a[u] = x[i + u * 32 * NW];
        t[u] = ld_cg(tmp + i + u * 32 * NW);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) x[i + u * 32 * NW] = a[u] - t[u];
    }
    for (; i < i1; i += 32 * NW) x[i] = x[i] - ld_cg(tmp + i);
  }
  }                                                                // (compute warps)
  if constexpr (SPLIT) cluster_sync_all();                         // no CTA leaves while a neighbour may still write
}

// Right-hand sides of k_tri_reg's L sweep in packed order (index = slice·32 + lane).
// DOWN: gather form dst[p] = src[lrow[p]] — coalesced writes, the reads hit L2
// (the input vector was just written).  UP: only the rows with F_l entries,
// dst[fpos[i]] = (F_l y_J)_{frow[i]} (~10 % of the rows at level 0); the other
// positions of the UP buffer are zero from setup on.
template <typename T>
__global__ void __launch_bounds__(256) k_pack_gather(int64_t np, const int *__restrict__ lrow, const T *__restrict__ src,
                                                     T *__restrict__ dst, const int *__restrict__ done,
                                                     int64_t lds = 0, int64_t ldd = 0) {
  // the packing map (setup data) is loaded before griddepcontrol.wait, while the
  // predecessor runs; after it only the gathers (PG positions per thread in flight)
#ifndef PACK_GATHER_PREFETCH
#define PACK_GATHER_PREFETCH 0   // measured: the prefetch form 0.965 vs 0.958 ms per C5 iteration
#endif
#if !PACK_GATHER_PREFETCH
  pdl_launch();
  pdl_wait();
  if (done && *done) return;
  src += (size_t)blockIdx.y * lds;
  dst += (size_t)blockIdx.y * ldd;
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < np; p += (int64_t)gridDim.x * blockDim.x) {
    const int r = lrow[p];
    dst[p] = r >= 0 ? src[r] : dzero<T>();
  }
  return;
#endif
  constexpr int PG = 16;
  pdl_launch();
  src += (size_t)blockIdx.y * lds;                                 // column blockIdx.y (several right-hand sides)
  dst += (size_t)blockIdx.y * ldd;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x, p0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int r[PG];
#pragma unroll
  for (int u = 0; u < PG; ++u) r[u] = p0 + u * stride < np ? lrow[p0 + u * stride] : -1;
  pdl_wait();
  if (done && *done) return;
  T v[PG];
#pragma unroll
  for (int u = 0; u < PG; ++u) v[u] = r[u] >= 0 ? src[r[u]] : dzero<T>();
#pragma unroll
  for (int u = 0; u < PG; ++u)
    if (p0 + u * stride < np) dst[p0 + u * stride] = v[u];
  for (int64_t p = p0 + PG * stride; p < np; p += stride) {        // (more than PG per thread)
    const int rr = lrow[p];
    dst[p] = rr >= 0 ? src[rr] : dzero<T>();
  }
}
template <typename T>
__global__ void __launch_bounds__(256) k_pack_f(int64_t nf, const int *__restrict__ fpos, const int *__restrict__ frow,
                                                const int64_t *__restrict__ Fptr, const int32_t *__restrict__ Fcol,
                                                const T *__restrict__ Fval, const T *__restrict__ y, int64_t nloc,
                                                const T *__restrict__ yh, int64_t nh, const T *__restrict__ yl,
                                                T *__restrict__ dst, const int *__restrict__ done, int64_t ldy = 0,
                                                int64_t ldd = 0, int64_t npu = 0, const int *__restrict__ urow = nullptr,
                                                T *__restrict__ xu = nullptr) {
  // F_l's structure for this thread's first row (setup data) is loaded before
  // griddepcontrol.wait; after it only the y gathers
  constexpr int EM = 8;
  pdl_launch();
  const int64_t stride = (int64_t)gridDim.x * blockDim.x, i0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const bool have = i0 < nf;
  const int pos0 = have ? fpos[i0] : 0, li0 = have ? frow[i0] : 0;
  const int64_t q0 = have ? Fptr[li0] : 0, q1 = have ? Fptr[li0 + 1] : 0;
  int32_t fc[EM];
  T fv[EM];
#pragma unroll
  for (int u = 0; u < EM; ++u) {
    fc[u] = q0 + u < q1 ? Fcol[q0 + u] : 0;
    fv[u] = q0 + u < q1 ? Fval[q0 + u] : dzero<T>();
  }
  pdl_wait();
  if (done && *done) return;
  y += (size_t)blockIdx.y * ldy;                                   // column blockIdx.y (one GPU: no halo / yl)
  dst += (size_t)blockIdx.y * ldd;
  // the level's current values x[rows] in U-packed order (k_tri_reg UP writes
  // x[row] = xu - U^-1 L^-1 F y in place; one column)
  for (int64_t p = i0; p < npu; p += stride) {
    const int r = urow[p];
    xu[p] = r >= 0 ? y[r] : dzero<T>();
  }
  auto g = [&](int64_t c) { return c < nloc ? y[c] : (c < nloc + nh ? yh[c - nloc] : yl[c - nloc - nh]); };
  if (have) {                                                      // the same p order as csr_dot
    T xg[EM], v = dzero<T>();
#pragma unroll
    for (int u = 0; u < EM; ++u) xg[u] = q0 + u < q1 ? g(fc[u]) : dzero<T>();
#pragma unroll
    for (int u = 0; u < EM; ++u)
      if (q0 + u < q1) v += fv[u] * xg[u];
    if (q1 - q0 > EM) v += csr_dot(q0 + EM, q1, Fcol, Fval, g);  // (long rows: the rest, in order)
    dst[pos0] = v;
  }
  for (int64_t i = i0 + stride; i < nf; i += stride) {
    const int li = frow[i];
    dst[fpos[i]] = csr_dot(Fptr[li], Fptr[li + 1], Fcol, Fval, g);
  }
}

// Packs the L-sweep right-hand sides of a stage in chunk order:
// DOWN: dst[lpos[i]] = src[row0 + i];  UP: dst[lpos[i]] = (F_l y_J)_{row0 + i},
// with F_l's columns local (< nloc), in the halo yh (< nloc + nh) or in the
// replicated last-separator vector yl.
template <typename T>
__global__ void __launch_bounds__(256) k_pack_rhs(int64_t nrows, int64_t row0, const int *__restrict__ lpos, T *__restrict__ dst,
                                                  const T *__restrict__ src, const int64_t *__restrict__ Fptr,
                                                  const int32_t *__restrict__ Fcol, const T *__restrict__ Fval,
                                                  int64_t Fbase, const T *__restrict__ y, int64_t nloc,
                                                  const T *__restrict__ yh, int64_t nh, const T *__restrict__ yl,
                                                  const int *__restrict__ done) {
  if (done && *done) return;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nrows; i += (int64_t)gridDim.x * blockDim.x) {
    T v;
    if (src) {
      v = src[row0 + i];
    } else {
      const int64_t li = row0 + i - Fbase;
      v = dzero<T>();
      for (int64_t p = Fptr[li]; p < Fptr[li + 1]; ++p) {
        const int64_t c = Fcol[p];
        const T yc = c < nloc ? y[c] : (c < nloc + nh ? yh[c - nloc] : yl[c - nloc - nh]);
        v += Fval[p] * yc;
      }
    }
    dst[lpos ? lpos[i] : row0 + i] = v;
  }
}

// Deterministic last-CTA reduction of per-CTA partials stored column-major
// (partial[c * G + q], q = CTA): warp w sums the columns w, w+8, ...; lane l
// adds the CTAs l, l+32, ... (coalesced, fixed order), then a fixed shuffle tree.
// The loads of a column (up to 16 per lane) are all issued before the sum, so
// a column costs one L2 round trip (the tail of every CGS2 pass with dots).
template <typename T>
__device__ inline void reduce_partials(const T *partial, int G, int ncol, T *out) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int c = warp; c < ncol; c += nw) {
    T s = dzero<T>();
    const T *p = partial + (int64_t)c * G;
    int q0 = 0;
    for (; q0 < G; q0 += 512) {
      T v[16];
#pragma unroll
      for (int u = 0; u < 16; ++u) {
        const int q = q0 + lane + 32 * u;
        v[u] = q < G ? ld_cg(p + q) : dzero<T>();
      }
#pragma unroll
      for (int u = 0; u < 16; ++u) s += v[u];
    }
    s = warp_sum(s);
    if (lane == 0) out[c] = s;
  }
}

// ----------------------------------------------------------------- K6+K7
// Rows J_l = [rowbase, rowbase + s): dst_i = src_i - Σ_j E_ij z_j (src == nullptr: 0;
// columns >= nloc in the halo zh), then per-column partial sums of conj(W_ic) dst_i;
// the last CTA reduces the partials in CTA order into this rank's part of
// s = W^H r_J (summed over ranks by an all-reduce).
// CTA = 8 warps; a tile is 256 rows; warp w owns the columns c ≡ w (mod 8).
// NACC accumulators per warp: k <= 8 NACC (instances 1, 2, 3, 4, 6, 8: k <= 64,
// chosen per level by ew_nacc on the host; the rank check of gemslr_setup keeps k <= 52).
constexpr int EW_MAXK = 64;
template <typename T, int NACC>
__global__ void __launch_bounds__(256) k_ew(int64_t s, int64_t rowbase, const int64_t *__restrict__ Eptr,
                                            const int32_t *__restrict__ Ecol, const T *__restrict__ Eval,
                                            const T *__restrict__ z, const T *__restrict__ zh, int64_t nloc,
                                            const T *src, T *dst, const T *__restrict__ W,
                                            int64_t ldw, int k, T *__restrict__ partial, unsigned *ticket,
                                            T *__restrict__ sout, const int *__restrict__ done) {
  if (done && *done) return;
  __shared__ T sv[256];
  __shared__ bool amlast;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  T acc[NACC];
#pragma unroll
  for (int a = 0; a < NACC; ++a) acc[a] = dzero<T>();
  const int64_t ntiles = (s + 255) / 256;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t i = tile * 256 + tid;
    T v = dzero<T>();
    if (i < s) {
      const T e = csr_dot(Eptr[i], Eptr[i + 1], Ecol, Eval,
                          [&](int64_t c) { return c < nloc ? z[c] : zh[c - nloc]; });
      v = (src ? src[rowbase + i] : dzero<T>()) - e;
      dst[rowbase + i] = v;
    }
    if (k > 0) {
      sv[tid] = v;
      __syncthreads();
#pragma unroll
      for (int a = 0; a < NACC; ++a) {
        const int c = warp + 8 * a;
        if (c < k) {
#pragma unroll
          for (int rr = 0; rr < 8; ++rr) {
            const int64_t ii = tile * 256 + rr * 32 + lane;
            if (ii < s) acc[a] += dconj(W[c * ldw + ii]) * sv[rr * 32 + lane];
          }
        }
      }
      __syncthreads();
    }
  }
  if (k == 0) return;
#pragma unroll
  for (int a = 0; a < NACC; ++a) {
    const int c = warp + 8 * a;
    T r = warp_sum(acc[a]);
    if (lane == 0 && c < k) partial[(int64_t)c * gridDim.x + blockIdx.x] = r;
  }
  __threadfence();
  __syncthreads();
  if (tid == 0) amlast = (atomicAdd(ticket, 1u) == gridDim.x - 1);
  __syncthreads();
  if (!amlast) return;
  __threadfence();
  reduce_partials(partial, (int)gridDim.x, k, sout);             // this rank's part of s = W^H r_J
  if (tid == 0) *ticket = 0;
}

// ----------------------------------------------------------------- K6+K7+K8 fused (one GPU)
// r_J = src_J - E_l z1 ; s = W_l^H r_J ; t = G_l s ; r_J += W_l t in ONE
// cooperative launch: the last CTA to finish the W^H partials reduces them in
// CTA order, forms t = G_l s and publishes it with a release flag
// (epoch); every CTA waits for it (all CTAs are co-resident) and adds W_l t to
// its rows.  Saves the second launch and its tail on the latency-bound levels.
// The flag is a generation counter in device memory: every CTA reads it before
// taking its ticket, the last CTA (which takes the final ticket, so after every
// read) advances it — no host-side epoch, so the launch can live in a CUDA graph.
#ifndef EW_UNROLL_WT
#define EW_UNROLL_WT 0
#endif
template <typename T, int NACC>
__global__ void __launch_bounds__(256) k_ewx(int64_t s, int64_t rowbase, const int64_t *__restrict__ Eptr,
                                             const int32_t *__restrict__ Ecol, const T *__restrict__ Eval,
                                             const T *__restrict__ z, const T *__restrict__ zh, int64_t nloc,
                                             const T *src, T *dst, const T *__restrict__ W, int64_t ldw, int k,
                                             const T *__restrict__ G, T *__restrict__ partial, unsigned *ticket,
                                             T *sout, int *flag, const int *__restrict__ done, int64_t npk = 0,
                                             const int *__restrict__ pkpos = nullptr, T *__restrict__ pk = nullptr) {
  pdl_launch();
  pdl_wait();
  if (done && *done) return;
  __shared__ T sv[256];
  __shared__ T st[64];
  __shared__ bool amlast;
  __shared__ int gen0;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  T acc[NACC];
#pragma unroll
  for (int a = 0; a < NACC; ++a) acc[a] = dzero<T>();
  const int64_t ntiles = (s + 255) / 256;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t i = tile * 256 + tid;
    T v = dzero<T>();
    if (i < s) {
      const T e = csr_dot(Eptr[i], Eptr[i + 1], Ecol, Eval,
                          [&](int64_t c) { return c < nloc ? z[c] : zh[c - nloc]; });
      v = (src ? src[rowbase + i] : dzero<T>()) - e;
      dst[rowbase + i] = v;
    }
    sv[tid] = v;
    __syncthreads();
#pragma unroll
    for (int a = 0; a < NACC; ++a) {
      const int c = warp + 8 * a;
      if (c < k) {
#pragma unroll
        for (int rr = 0; rr < 8; ++rr) {
          const int64_t ii = tile * 256 + rr * 32 + lane;
          if (ii < s) acc[a] += dconj(W[c * ldw + ii]) * sv[rr * 32 + lane];
        }
      }
    }
    __syncthreads();
  }
#pragma unroll
  for (int a = 0; a < NACC; ++a) {
    const int c = warp + 8 * a;
    T r = warp_sum(acc[a]);
    if (lane == 0 && c < k) partial[(int64_t)c * gridDim.x + blockIdx.x] = r;
  }
  __threadfence();
  __syncthreads();
  if (tid == 0) {
    int g;
    asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(g) : "l"(flag) : "memory");
    gen0 = g;
    amlast = (atomicAdd(ticket, 1u) == gridDim.x - 1);
  }
  __syncthreads();
  const int epoch = gen0 + 1;
  if (amlast) {
    __threadfence();
    reduce_partials(partial, (int)gridDim.x, k, sout);             // s = W^H r_J
    __syncthreads();
    if (tid < k) {                                                 // t = G s
      T t = dzero<T>();
#pragma unroll
      for (int a = 0; a < 8 * NACC; ++a)                           // all loads in flight (a loop over k was
        if (a < k) t += G[(int64_t)a * k + tid] * ld_cg(sout + a); // k dependent L2 round trips)
      sout[64 + tid] = t;
    }
    __threadfence();
    __syncthreads();
    if (tid == 0) {
      *ticket = 0;
      asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(flag), "r"(epoch) : "memory");
    }
  }
  if (tid == 0) {
    int f;
    do {
      asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(f) : "l"(flag) : "memory");
      if (f != epoch) __nanosleep(64);
    } while (f != epoch);
  }
  __syncthreads();
  if (tid < k) st[tid] = ld_cg(sout + 64 + tid);
  __syncthreads();
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {  // r_J += W t
    const int64_t i = tile * 256 + tid;
    if (i < s) {
      T a = dzero<T>();
#if EW_UNROLL_WT
#pragma unroll
      for (int c = 0; c < 8 * NACC; ++c)
        if (c < k) a += ld_nc(W + c * ldw + i) * st[c];
#else
      for (int c = 0; c < k; ++c) a += ld_nc(W + c * ldw + i) * st[c];
#endif
      const T v = ld_cg(dst + rowbase + i) + a;
      dst[rowbase + i] = v;
      if (i < npk) pk[pkpos[i]] = v;                               // the next stage's packed right-hand side
    }
  }
}

// ----------------------------------------------------------------- K6+K7+K8 on one cluster (small s_l)
// The same as k_ewx for the small interfaces of the deeper levels (C5: s_1 = 4.6k,
// s_2 = 667 rows), where a grid-wide hand-off costs more than the work: ONE
// cluster of C CTAs, CTA c owns the rows [c s / C, (c+1) s / C).  Each CTA sums
// its W^H r_J partials over its warps (fixed order) into shared memory; after a
// cluster barrier every CTA reads the C partial vectors through DSMEM in rank
// order (the same s in all CTAs), forms t = G s and adds W t to its rows; a second
// cluster barrier keeps the partials alive until every CTA has read them.
__device__ inline double ld_dsmem(unsigned addr, double) {
  double v;
  asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(v) : "r"(addr));
  return v;
}
__device__ inline cd ld_dsmem(unsigned addr, cd) {
  cd v;
  asm volatile("ld.shared::cluster.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(addr));
  return v;
}
template <typename T, int NACC>
__global__ void __launch_bounds__(256) k_ewc(int64_t s, int64_t rowbase, const int64_t *__restrict__ Eptr,
                                             const int32_t *__restrict__ Ecol, const T *__restrict__ Eval,
                                             const T *__restrict__ z, const T *__restrict__ zh, int64_t nloc,
                                             const T *src, T *dst, const T *__restrict__ W, int64_t ldw, int k,
                                             const T *__restrict__ G, const int *__restrict__ done, int64_t npk = 0,
                                             const int *__restrict__ pkpos = nullptr, T *__restrict__ pk = nullptr) {
  // One row per thread (s <= 256 C).  Everything that is setup data — the row's E
  // entries, its W row, G, its packed position — is loaded BEFORE griddepcontrol.wait,
  // while the predecessor still runs; after it only the z gathers and src remain,
  // then two cluster barriers.  (A tile loop with the loads after the wait made this
  // a chain of ~10 dependent memory round trips: 15-28 us for 667 / 4.6k rows.)
  constexpr int KM = 8 * NACC, EM = 8;
  pdl_launch();
  __shared__ T Gs[KM * KM];
  __shared__ T wpart[8][KM];
  __shared__ T cpart[KM];
  __shared__ T sv[KM], st[KM];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const unsigned C = gridDim.x, c = blockIdx.x;
  const int64_t r0 = s * c / C, r1 = s * (c + 1) / C;
  const int64_t i = r0 + tid;
  const bool own = i < r1;
  const int64_t p0 = own ? Eptr[i] : 0, p1 = own ? Eptr[i + 1] : 0;
  int32_t ec[EM];
  T ev[EM], wr[KM];
#pragma unroll
  for (int u = 0; u < EM; ++u) {
    ec[u] = p0 + u < p1 ? Ecol[p0 + u] : 0;
    ev[u] = p0 + u < p1 ? Eval[p0 + u] : dzero<T>();
  }
#pragma unroll
  for (int cc = 0; cc < KM; ++cc) wr[cc] = (own && cc < k) ? ld_nc(W + cc * ldw + i) : dzero<T>();
  for (int q = tid; q < k * k; q += blockDim.x) Gs[q] = G[q];
  const int ppk = (own && i < npk) ? pkpos[i] : -1;
  pdl_wait();
  if (done && *done) return;                                       // uniform over the cluster (predecessor complete)
  T v = dzero<T>();
  if (own) {
    auto g = [&](int64_t cc) { return cc < nloc ? z[cc] : zh[cc - nloc]; };
    T e = dzero<T>(), xg[EM];
#pragma unroll
    for (int u = 0; u < EM; ++u) xg[u] = p0 + u < p1 ? g(ec[u]) : dzero<T>();
#pragma unroll
    for (int u = 0; u < EM; ++u)
      if (p0 + u < p1) e += ev[u] * xg[u];
    for (int64_t p = p0 + EM; p < p1; ++p) e += Eval[p] * g(Ecol[p]);   // rows with more entries (rare)
    v = (src ? src[rowbase + i] : dzero<T>()) - e;
  }
#pragma unroll
  for (int cc = 0; cc < KM; ++cc) {                                // this CTA's part of W^H r_J
    if (cc < k) {
      const T r = warp_sum(dconj(wr[cc]) * v);
      if (lane == 0) wpart[warp][cc] = r;
    }
  }
  __syncthreads();
  if (tid < k) {
    T r = dzero<T>();
#pragma unroll
    for (int q = 0; q < 8; ++q) r += wpart[q][tid];
    cpart[tid] = r;
  }
  cluster_sync_all();
  if (tid < k) {                                                   // s over the cluster, rank order
    T sc = dzero<T>();
    const unsigned a0 = smem_u32(&cpart[tid]);
    for (unsigned q = 0; q < C; ++q) sc += ld_dsmem(mapa_shared(a0, q), dzero<T>());
    sv[tid] = sc;
  }
  __syncthreads();
  if (tid < k) {                                                   // t = G s
    T t = dzero<T>();
    for (int a = 0; a < k; ++a) t += Gs[a * k + tid] * sv[a];
    st[tid] = t;
  }
  __syncthreads();
  if (own) {                                                       // r_J += W t
    T a = dzero<T>();
#pragma unroll
    for (int cc = 0; cc < KM; ++cc)
      if (cc < k) a += wr[cc] * st[cc];
    const T v2 = v + a;
    dst[rowbase + i] = v2;
    if (ppk >= 0) pk[ppk] = v2;                                    // the next stage's packed right-hand side
  }
  cluster_sync_all();                                              // partials read by every CTA before any exits
}

// ----------------------------------------------------------------- K6+K7+K8 for large s_l (PDL, grid barrier)
// The same one-row-per-thread form as k_ewc for the large interfaces (C5 s_0 = 113k,
// s_1 = 4.6k), launched with programmatic dependent launch instead of as a
// cooperative kernel: the setup data of every row (its E entries, its W row, G,
// its packed position) is loaded while the predecessor trisolve still runs; after
// griddepcontrol.wait: the z gathers, this CTA's partial of W^H r_J, a grid barrier
// (a per-call-site ticket counter: this launch's CTAs wait for the round of
// gridDim.x tickets to complete), every CTA sums all partials in CTA order (the same
// s everywhere, deterministic), t = G s, r_J += W t.  griddepcontrol.launch_dependents
// is issued only after the barrier, so no successor CTA can take an SM while a CTA
// of this grid still waits to become resident (the host checks that the grid fits
// the SMs at the occupancy of this kernel, else it uses k_ewx).
template <typename T, int NACC>
__global__ void __launch_bounds__(256, 3) k_ewg(int64_t s, int64_t rowbase, const int64_t *__restrict__ Eptr,
                                                const int32_t *__restrict__ Ecol, const T *__restrict__ Eval,
                                                const T *__restrict__ z, const T *__restrict__ zh, int64_t nloc,
                                                const T *src, T *dst, const T *__restrict__ W, int64_t ldw, int k,
                                                const T *__restrict__ G, T *__restrict__ partial,
                                                unsigned *__restrict__ ticket, const int *__restrict__ done,
                                                int64_t npk = 0, const int *__restrict__ pkpos = nullptr,
                                                T *__restrict__ pk = nullptr) {
  constexpr int KM = 8 * NACC, EM = 4;
  __shared__ T Gs[KM * KM];
  __shared__ T wpart[8][KM];
  __shared__ T sv[KM], st[KM];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t i = (int64_t)blockIdx.x * 256 + tid;
  const bool own = i < s;
  const int64_t p0 = own ? Eptr[i] : 0, p1 = own ? Eptr[i + 1] : 0;
  int32_t ec[EM];
  T ev[EM], wr[KM];
#pragma unroll
  for (int u = 0; u < EM; ++u) {
    ec[u] = p0 + u < p1 ? Ecol[p0 + u] : 0;
    ev[u] = p0 + u < p1 ? Eval[p0 + u] : dzero<T>();
  }
#pragma unroll
  for (int cc = 0; cc < KM; ++cc) wr[cc] = (own && cc < k) ? ld_nc(W + cc * ldw + i) : dzero<T>();
  for (int q = tid; q < k * k; q += blockDim.x) Gs[q] = G[q];
  const int ppk = (own && i < npk) ? pkpos[i] : -1;
  pdl_wait();
  if (done && *done) return;                                       // uniform over the grid (predecessor complete)
  T v = dzero<T>();
  if (own) {
    auto g = [&](int64_t cc) { return cc < nloc ? z[cc] : zh[cc - nloc]; };
    T e = dzero<T>(), xg[EM];
#pragma unroll
    for (int u = 0; u < EM; ++u) xg[u] = p0 + u < p1 ? g(ec[u]) : dzero<T>();
#pragma unroll
    for (int u = 0; u < EM; ++u)
      if (p0 + u < p1) e += ev[u] * xg[u];
    for (int64_t p = p0 + EM; p < p1; ++p) e += Eval[p] * g(Ecol[p]);   // rows with more entries
    v = (src ? src[rowbase + i] : dzero<T>()) - e;
  }
#pragma unroll
  for (int cc = 0; cc < KM; ++cc) {
    if (cc < k) {
      const T r = warp_sum(dconj(wr[cc]) * v);
      if (lane == 0) wpart[warp][cc] = r;
    }
  }
  __syncthreads();
  const unsigned Gn = gridDim.x;
  if (tid < k) {
    T r = dzero<T>();
#pragma unroll
    for (int q = 0; q < 8; ++q) r += wpart[q][tid];
    partial[(int64_t)tid * Gn + blockIdx.x] = r;
  }
  __threadfence();
  __syncthreads();
  if (tid == 0) {                                                  // grid barrier: this launch's round of tickets
    const unsigned t = atomicAdd(ticket, 1u);
    const unsigned end = (t / Gn + 1) * Gn;
    unsigned c;
    do {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(c) : "l"(ticket) : "memory");
    } while ((int)(c - end) < 0);
  }
  __syncthreads();
  pdl_launch();
  // s = sum over the CTAs of the partials, in CTA order (the same in every CTA)
  for (int cc = warp; cc < k; cc += 8) {
    const T *pp = partial + (int64_t)cc * Gn;
    T a = dzero<T>();
    for (unsigned q0 = 0; q0 < Gn; q0 += 256) {
      T vv[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const unsigned q = q0 + lane + 32 * u;
        vv[u] = q < Gn ? ld_cg(pp + q) : dzero<T>();
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) a += vv[u];
    }
    a = warp_sum(a);
    if (lane == 0) sv[cc] = a;
  }
  __syncthreads();
  if (tid < k) {                                                   // t = G s
    T t = dzero<T>();
    for (int a = 0; a < k; ++a) t += Gs[a * k + tid] * sv[a];
    st[tid] = t;
  }
  __syncthreads();
  if (own) {                                                       // r_J += W t
    T a = dzero<T>();
#pragma unroll
    for (int cc = 0; cc < KM; ++cc)
      if (cc < k) a += wr[cc] * st[cc];
    const T v2 = v + a;
    dst[rowbase + i] = v2;
    if (ppk >= 0) pk[ppk] = v2;                                    // the next stage's packed right-hand side
  }
}

// ----------------------------------------------------------------- K8
// r_J += W_l (G_l s): the k x k product G_l s is formed redundantly by every
// CTA in its prologue, G_l column-major.
template <typename T>
__global__ void __launch_bounds__(256) k_waxpy(int64_t s, int64_t rowbase, const T *__restrict__ W, int64_t ldw, int k,
                                               const T *__restrict__ G, const T *__restrict__ sv, T *dst,
                                               const int *__restrict__ done, int64_t npk = 0,
                                               const int *__restrict__ pkpos = nullptr, T *__restrict__ pk = nullptr) {
  if (done && *done) return;
  __shared__ T ss[64], st[64];
  if (threadIdx.x < k) ss[threadIdx.x] = sv[threadIdx.x];
  __syncthreads();
  if (threadIdx.x < k) {
    T t = dzero<T>();
#pragma unroll 8
    for (int a = 0; a < k; ++a) t += G[(int64_t)a * k + threadIdx.x] * ss[a];
    st[threadIdx.x] = t;
  }
  __syncthreads();
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < s; i += (int64_t)gridDim.x * blockDim.x) {
    T acc = dzero<T>();
#pragma unroll 8
    for (int c = 0; c < k; ++c) acc += ld_nc(W + c * ldw + i) * st[c];
    const T v = dst[rowbase + i] + acc;
    dst[rowbase + i] = v;
    if (i < npk) pk[pkpos[i]] = v;                                 // the next stage's packed right-hand side
  }
}

// ----------------------------------------------------------------- K10-K12 CGS2
// V column-major (ld), ncols <= GS_MAXC.  A CTA of 8 warps walks 32-row tiles;
// warp w owns the columns c ≡ w (mod 8) and keeps those V values of the tile
// in registers for the update and the dot of the same pass.
//   pass 1 (upd = 0, dot = 1): res = [V^H w, ||w||^2]
//   pass 2 (upd = 1, dot = 1): w -= V h_in ; res = [V^H w, ||w||^2]
//   pass 3 (upd = 1, dot = 0): w -= V h_in ; res = [||w||^2]
// Results are reduced in fixed CTA order by the last CTA (ticket).
// A step covers TR 32-row tiles; warp w owns the columns w + 8a, a < NPW, with
// TR * NPW <= 13 values of V in registers (instances chosen by ncols so the
// loads in flight per thread stay ~13 however many columns there are).
constexpr int GS_MAXC = 104;               // >= restart + 1
template <typename T, int TR, int NPW>
__global__ void __launch_bounds__(256) k_gs(int64_t n, const T *__restrict__ V, int64_t ldv, int ncols, T *w, int upd,
                                            int dot, const T *__restrict__ h_in, T *__restrict__ partial,
                                            unsigned *ticket, T *__restrict__ res, const int *__restrict__ done) {
  pdl_launch();
  pdl_wait();
  if (done && *done) return;
  __shared__ T su[8][32 * TR];
  __shared__ T sh[GS_MAXC];
  __shared__ bool amlast;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (upd)
    for (int c = tid; c < ncols; c += blockDim.x) sh[c] = h_in[c];
  __syncthreads();
  T acc[NPW];
#pragma unroll
  for (int a = 0; a < NPW; ++a) acc[a] = dzero<T>();
  double nrm = 0.0;
  const int64_t nsteps = (n + 32 * TR - 1) / (32 * TR);
  for (int64_t step = blockIdx.x; step < nsteps; step += gridDim.x) {
    const int64_t base = step * 32 * TR + lane;
    T vr[TR][NPW];
    T wi[TR];
#pragma unroll
    for (int r = 0; r < TR; ++r) {
      const int64_t i = base + 32 * r;
      const bool ok = i < n;
#pragma unroll
      for (int a = 0; a < NPW; ++a) {
        const int c = warp + 8 * a;
        vr[r][a] = (ok && c < ncols) ? ld_nc(V + c * ldv + i) : dzero<T>();
      }
      wi[r] = ok ? w[i] : dzero<T>();
    }
    if (upd) {
#pragma unroll
      for (int r = 0; r < TR; ++r) {
        T u = dzero<T>();
#pragma unroll
        for (int a = 0; a < NPW; ++a) {
          const int c = warp + 8 * a;
          if (c < ncols) u += vr[r][a] * sh[c];
        }
        su[warp][r * 32 + lane] = u;
      }
      __syncthreads();
#pragma unroll
      for (int r = 0; r < TR; ++r) {
        T tot = dzero<T>();
#pragma unroll
        for (int q = 0; q < 8; ++q) tot += su[q][r * 32 + lane];
        wi[r] = wi[r] - tot;
      }
      __syncthreads();
      if (warp == 0)
#pragma unroll
        for (int r = 0; r < TR; ++r)
          if (base + 32 * r < n) w[base + 32 * r] = wi[r];
    }
    if (dot) {
#pragma unroll
      for (int r = 0; r < TR; ++r)
#pragma unroll
        for (int a = 0; a < NPW; ++a) acc[a] += dconj(vr[r][a]) * wi[r];
    }
    if (warp == 0)
#pragma unroll
      for (int r = 0; r < TR; ++r) nrm += dabs2(wi[r]);
  }
  // per-warp reduction; warp w owns its columns, warp 0 owns the norm
  const int nres = dot ? ncols + 1 : 1;
  if (dot) {
#pragma unroll
    for (int a = 0; a < NPW; ++a) {
      const int c = warp + 8 * a;
      T r = warp_sum(acc[a]);
      if (lane == 0 && c < ncols) partial[(int64_t)c * gridDim.x + blockIdx.x] = r;
    }
  }
  if (warp == 0) {
    double r = warp_sum(nrm);
    if (lane == 0) {
      T t = dzero<T>();
      if constexpr (sizeof(T) == sizeof(double)) t = r; else t = T{r, 0.0};
      partial[(int64_t)(nres - 1) * gridDim.x + blockIdx.x] = t;
    }
  }
  __threadfence();
  __syncthreads();
  if (tid == 0) amlast = (atomicAdd(ticket, 1u) == gridDim.x - 1);
  __syncthreads();
  if (!amlast) return;
  __threadfence();
  reduce_partials(partial, (int)gridDim.x, nres, res);
  if (tid == 0) *ticket = 0;
}

// Warp-tile form of the CGS2 passes: a warp owns 32-row tiles and ALL columns
// (NC >= ncols, the tile's V values stay in registers between the update and
// the dot), so there is no block barrier per tile.  The dots of a tile are
// reduced over the lanes by a transpose-butterfly (31 shuffles per 32 columns;
// afterwards lane i holds column i), accumulated in registers, and reduced over
// the warps and CTAs once at the end (deterministic, fixed order).
template <typename T>
__device__ inline T shfl_x(T v, int m) { return shfl_xor(v, m); }
template <typename T>
__device__ inline void tbfly32(T (&x)[32], int lane) {              // lane i <- sum over lanes of x[i]
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) {
    const bool up = (lane & o) != 0;
#pragma unroll
    for (int k = 0; k < o; ++k) {
      const T send = up ? x[k] : x[k + o];
      const T keep = up ? x[k + o] : x[k];
      x[k] = keep + shfl_x(send, o);
    }
  }
}
// TU tiles per warp iteration (their loads all in flight: with few columns one
// tile is too little memory-level parallelism — k_gs2<8> ran at 0.7-3 TB/s with
// TU = 1).  LA: the dots are accumulated per lane over all of the warp's tiles
// and reduced over the lanes once at the end (NC <= 16, registers allow); else
// the transpose butterfly per TU tiles.
template <typename T, int NC, int TU = 1, bool LA = false>
__global__ void __launch_bounds__(256, NC * TU * sizeof(T) > 256 ? 1 : 2) k_gs2(int64_t n, const T *__restrict__ V, int64_t ldv, int ncols, T *w, int upd,
                                              int dot, const T *__restrict__ h_in, T *__restrict__ partial,
                                              unsigned *ticket, T *__restrict__ res, const int *__restrict__ done) {
  pdl_launch();
  pdl_wait();
  if (done && *done) return;
  constexpr int NCH = LA ? 0 : (NC + 31) / 32;                     // 32-column butterfly chunks
  constexpr int NA = LA ? NC : 1;                                  // per-lane accumulators
  __shared__ T sh[NC];
  __shared__ T red[8][NC + 1];
  __shared__ bool amlast;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int c = tid; c < NC; c += blockDim.x) sh[c] = (upd && c < ncols) ? h_in[c] : dzero<T>();
  __syncthreads();
  T acc[NCH > 0 ? NCH : 1];
#pragma unroll
  for (int q = 0; q < (NCH > 0 ? NCH : 1); ++q) acc[q] = dzero<T>();
  T la[NA];
#pragma unroll
  for (int c = 0; c < NA; ++c) la[c] = dzero<T>();
  double nrm = 0.0;
  const int64_t ntiles = (n + 31) / 32;
  for (int64_t t0 = ((int64_t)blockIdx.x * 8 + warp) * TU; t0 < ntiles; t0 += (int64_t)gridDim.x * 8 * TU) {
    T v[TU][NC], wi[TU];
#pragma unroll
    for (int u = 0; u < TU; ++u) {
      const int64_t r = (t0 + u) * 32 + lane;
      const bool ok = r < n;
#pragma unroll
      for (int c = 0; c < NC; ++c) v[u][c] = (c < ncols && ok) ? ld_nc(V + c * ldv + r) : dzero<T>();
      wi[u] = ok ? w[r] : dzero<T>();
    }
#pragma unroll
    for (int u = 0; u < TU; ++u) {
      const int64_t r = (t0 + u) * 32 + lane;
      if (upd) {
        T u0 = dzero<T>(), u1 = dzero<T>();
#pragma unroll
        for (int c = 0; c < NC; c += 2) {
          u0 += v[u][c] * sh[c];
          if (c + 1 < NC) u1 += v[u][c + 1 < NC ? c + 1 : 0] * sh[c + 1 < NC ? c + 1 : 0];
        }
        wi[u] = wi[u] - (u0 + u1);
        if (r < n) w[r] = wi[u];
      }
      nrm += dabs2(wi[u]);
    }
    if (dot) {
      if constexpr (LA) {
#pragma unroll
        for (int u = 0; u < TU; ++u)
#pragma unroll
          for (int c = 0; c < NC; ++c) la[c] += dconj(v[u][c]) * wi[u];
      } else {
#pragma unroll
        for (int q = 0; q < NCH; ++q) {
          T x[32];
#pragma unroll
          for (int k = 0; k < 32; ++k) {
            const int c = 32 * q + k < NC ? 32 * q + k : 0;
            T t = dzero<T>();
#pragma unroll
            for (int u = 0; u < TU; ++u) t += dconj(v[u][c]) * wi[u];
            x[k] = (32 * q + k < NC) ? t : dzero<T>();
          }
          tbfly32(x, lane);
          acc[q] += x[0];
        }
      }
    }
  }
  // lane i of warp w holds column 32 q + i of this warp (LA: every lane a part of
  // every column, summed over the lanes here); warp 0 the norm too
  const int nres = dot ? ncols + 1 : 1;
  nrm = warp_sum(nrm);
  if constexpr (LA) {
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      const T t = warp_sum(la[c]);
      if (lane == c) red[warp][c] = t;
    }
  } else {
#pragma unroll
    for (int q = 0; q < NCH; ++q)
      if (32 * q + lane < NC) red[warp][32 * q + lane] = acc[q];
  }
  if (lane == 0) {
    T t = dzero<T>();
    if constexpr (sizeof(T) == sizeof(double)) t = nrm; else t = T{nrm, 0.0};
    red[warp][NC] = t;
  }
  __syncthreads();
  for (int c = tid; c < nres; c += blockDim.x) {
    const int src = (c == nres - 1) ? NC : c;
    T t = dzero<T>();
#pragma unroll
    for (int q = 0; q < 8; ++q) t += red[q][src];
    partial[(int64_t)c * gridDim.x + blockIdx.x] = t;
  }
  __threadfence();
  __syncthreads();
  if (tid == 0) amlast = (atomicAdd(ticket, 1u) == gridDim.x - 1);
  __syncthreads();
  if (!amlast) return;
  __threadfence();
  reduce_partials(partial, (int)gridDim.x, nres, res);
  if (tid == 0) *ticket = 0;
}

// The same with 33..64 columns: a warp covers 16 rows, lanes 0-15 hold columns
// 0..31 and lanes 16-31 columns 32..63 of the same rows (32 values per lane as
// in k_gs2<T, 32>); the two halves of the update are combined with one
// shuffle and the dots reduced over the 16 lanes of a half (15 shuffles per 16
// columns; afterwards lane sub of half h holds columns 32h + sub and 32h + 16 + sub).
template <typename T>
__device__ inline void tbfly16(T (&x)[16], int sub) {
#pragma unroll
  for (int o = 8; o >= 1; o >>= 1) {
    const bool up = (sub & o) != 0;
#pragma unroll
    for (int k = 0; k < o; ++k) {
      const T send = up ? x[k] : x[k + o];
      const T keep = up ? x[k + o] : x[k];
      x[k] = keep + shfl_x(send, o);
    }
  }
}
template <typename T>
__global__ void __launch_bounds__(256, 2) k_gs2h(int64_t n, const T *__restrict__ V, int64_t ldv, int ncols, T *w, int upd,
                                               int dot, const T *__restrict__ h_in, T *__restrict__ partial,
                                               unsigned *ticket, T *__restrict__ res, const int *__restrict__ done) {
  pdl_launch();
  pdl_wait();
  if (done && *done) return;
  __shared__ T sh[64];
  __shared__ T red[8][65];
  __shared__ bool amlast;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int half = lane >> 4, sub = lane & 15;
  for (int c = tid; c < 64; c += blockDim.x) sh[c] = (upd && c < ncols) ? h_in[c] : dzero<T>();
  __syncthreads();
  T acc0 = dzero<T>(), acc1 = dzero<T>();
  double nrm = 0.0;
  const int64_t ntiles = (n + 15) / 16;
  const T *Vh = V + (int64_t)(32 * half) * ldv;
  const int nc = ncols - 32 * half;                                 // columns of this half
  for (int64_t tile = (int64_t)blockIdx.x * 8 + warp; tile < ntiles; tile += (int64_t)gridDim.x * 8) {
    const int64_t r = tile * 16 + sub;
    const bool ok = r < n;
    T v[32];
#pragma unroll
    for (int k = 0; k < 32; ++k) v[k] = (k < nc && ok) ? ld_nc(Vh + k * ldv + r) : dzero<T>();
    T wi = ok ? w[r] : dzero<T>();
    if (upd) {
      T u0 = dzero<T>(), u1 = dzero<T>();
#pragma unroll
      for (int k = 0; k < 32; k += 2) {
        u0 += v[k] * sh[32 * half + k];
        u1 += v[k + 1] * sh[32 * half + k + 1];
      }
      T u = u0 + u1;
      u = u + shfl_x(u, 16);
      wi = wi - u;
      if (ok && half == 0) w[r] = wi;
    }
    if (half == 0) nrm += dabs2(wi);
    if (dot) {
      T x[16];
#pragma unroll
      for (int k = 0; k < 16; ++k) x[k] = dconj(v[k]) * wi;
      tbfly16(x, sub);
      acc0 += x[0];
#pragma unroll
      for (int k = 0; k < 16; ++k) x[k] = dconj(v[16 + k]) * wi;
      tbfly16(x, sub);
      acc1 += x[0];
    }
  }
  const int nres = dot ? ncols + 1 : 1;
  nrm = warp_sum(nrm);
  red[warp][32 * half + sub] = acc0;
  red[warp][32 * half + 16 + sub] = acc1;
  if (lane == 0) {
    T t = dzero<T>();
    if constexpr (sizeof(T) == sizeof(double)) t = nrm; else t = T{nrm, 0.0};
    red[warp][64] = t;
  }
  __syncthreads();
  for (int c = tid; c < nres; c += blockDim.x) {
    const int src = (c == nres - 1) ? 64 : c;
    T t = dzero<T>();
#pragma unroll
    for (int q = 0; q < 8; ++q) t += red[q][src];
    partial[(int64_t)c * gridDim.x + blockIdx.x] = t;
  }
  __threadfence();
  __syncthreads();
  if (tid == 0) amlast = (atomicAdd(ticket, 1u) == gridDim.x - 1);
  __syncthreads();
  if (!amlast) return;
  __threadfence();
  reduce_partials(partial, (int)gridDim.x, nres, res);
  if (tid == 0) *ticket = 0;
}

// Grouped warp tiles for many columns (complex restart-100 cycles): a warp covers
// RW = 32 / G rows; lane group g (RW lanes) holds columns [g*C, g*C + C) of those
// rows.  Update: partial sums combined over the groups by log2(G) shuffles; dot:
// per group a transpose-butterfly over its RW lanes (RW - 1 shuffles per RW
// columns; afterwards lane sub of group g holds column g*C + q*RW + sub).
template <int RW, typename T>
__device__ inline void tbfly_n(T (&x)[RW], int sub) {
#pragma unroll
  for (int o = RW / 2; o >= 1; o >>= 1) {
    const bool up = (sub & o) != 0;
#pragma unroll
    for (int k = 0; k < o; ++k) {
      const T send = up ? x[k] : x[k + o];
      const T keep = up ? x[k + o] : x[k];
      x[k] = keep + shfl_x(send, o);
    }
  }
}
template <typename T, int G, int C>
__global__ void __launch_bounds__(256, G >= 8 ? 2 : 1) k_gs2g(int64_t n, const T *__restrict__ V, int64_t ldv, int ncols, T *w, int upd,
                                                int dot, const T *__restrict__ h_in, T *__restrict__ partial,
                                                unsigned *ticket, T *__restrict__ res, const int *__restrict__ done) {
  pdl_launch();
  pdl_wait();
  if (done && *done) return;
  constexpr int RW = 32 / G, NQ = (C + RW - 1) / RW, NC = G * C;
  __shared__ T sh[NC];
  __shared__ T red[8][NC + 1];
  __shared__ bool amlast;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int grp = lane / RW, sub = lane % RW;
  for (int c = tid; c < NC; c += blockDim.x) sh[c] = (upd && c < ncols) ? h_in[c] : dzero<T>();
  __syncthreads();
  T acc[NQ];
#pragma unroll
  for (int q = 0; q < NQ; ++q) acc[q] = dzero<T>();
  double nrm = 0.0;
  const int64_t ntiles = (n + RW - 1) / RW;
  const T *Vg = V + (int64_t)(grp * C) * ldv;
  const int nc = ncols - grp * C;
  for (int64_t tile = (int64_t)blockIdx.x * 8 + warp; tile < ntiles; tile += (int64_t)gridDim.x * 8) {
    const int64_t r = tile * RW + sub;
    const bool ok = r < n;
    T v[C];
#pragma unroll
    for (int k = 0; k < C; ++k) v[k] = (k < nc && ok) ? ld_nc(Vg + k * ldv + r) : dzero<T>();
    T wi = ok ? w[r] : dzero<T>();
    if (upd) {
      T u0 = dzero<T>(), u1 = dzero<T>();
#pragma unroll
      for (int k = 0; k < C; k += 2) {
        u0 += v[k] * sh[grp * C + k];
        if (k + 1 < C) u1 += v[k + 1 < C ? k + 1 : 0] * sh[grp * C + (k + 1 < C ? k + 1 : 0)];
      }
      T u = u0 + u1;
#pragma unroll
      for (int o = RW; o < 32; o <<= 1) u = u + shfl_x(u, o);
      wi = wi - u;
      if (ok && grp == 0) w[r] = wi;
    }
    if (grp == 0) nrm += dabs2(wi);
    if (dot) {
#pragma unroll
      for (int q = 0; q < NQ; ++q) {
        T x[RW];
#pragma unroll
        for (int k = 0; k < RW; ++k) x[k] = (q * RW + k < C) ? dconj(v[q * RW + k < C ? q * RW + k : 0]) * wi : dzero<T>();
        tbfly_n<RW>(x, sub);
        acc[q] += x[0];
      }
    }
  }
  const int nres = dot ? ncols + 1 : 1;
  nrm = warp_sum(nrm);
#pragma unroll
  for (int q = 0; q < NQ; ++q)
    if (q * RW + sub < C) red[warp][grp * C + q * RW + sub] = acc[q];
  if (lane == 0) {
    T t = dzero<T>();
    if constexpr (sizeof(T) == sizeof(double)) t = nrm; else t = T{nrm, 0.0};
    red[warp][NC] = t;
  }
  __syncthreads();
  for (int c = tid; c < nres; c += blockDim.x) {
    const int src = (c == nres - 1) ? NC : c;
    T t = dzero<T>();
#pragma unroll
    for (int q = 0; q < 8; ++q) t += red[q][src];
    partial[(int64_t)c * gridDim.x + blockIdx.x] = t;
  }
  __threadfence();
  __syncthreads();
  if (tid == 0) amlast = (atomicAdd(ticket, 1u) == gridDim.x - 1);
  __syncthreads();
  if (!amlast) return;
  __threadfence();
  reduce_partials(partial, (int)gridDim.x, nres, res);
  if (tid == 0) *ticket = 0;
}

// ----------------------------------------------------------------- FGMRES column (1 thread)
template <typename T>
struct FgmDev {
  int *done;          // [0] done flag
  int *ints;          // [0] jend, [1] its, [2] maxit
  double *dbl;        // [0] bnorm, [1] rtol, [2] 1/H[j+1,j]
  double *hist;       // residual estimate history (maxit + 1)
  T *H;               // (m+1) x m column-major, rotated
  T *g;               // m + 1
  double *cs;         // m
  T *sn;              // m
};

template <typename T>
__device__ inline void fgmres_col_body(FgmDev<T> f, int m, int j, const T *__restrict__ res1, const T *__restrict__ res2,
                                       const T *__restrict__ res3) {
  T *Hj = f.H + (int64_t)j * (m + 1);
  double eta2, hn2;
  if constexpr (sizeof(T) == sizeof(double)) { eta2 = res1[j + 1]; hn2 = res3[0]; }
  else { eta2 = res1[j + 1].x; hn2 = res3[0].x; }
  const double eta = sqrt(eta2 > 0 ? eta2 : 0.0);
  const double hnext = sqrt(hn2 > 0 ? hn2 : 0.0);
  for (int i = 0; i <= j; ++i) Hj[i] = res1[i] + res2[i];
  if constexpr (sizeof(T) == sizeof(double)) Hj[j + 1] = hnext; else Hj[j + 1] = T{hnext, 0.0};
  for (int i = 0; i < j; ++i) {                       // previous rotations
    const T p = Hj[i], q = Hj[i + 1];
    Hj[i] = f.cs[i] * p + dconj(f.sn[i]) * q;
    Hj[i + 1] = (-f.sn[i]) * p + f.cs[i] * q;
  }
  const T a = Hj[j];
  const double aa = sqrt(dabs2(a)), bb = hnext;
  double c;
  T s;
  if (bb == 0.0) { c = 1.0; s = dzero<T>(); }
  else if (aa == 0.0) {
    c = 0.0;
    if constexpr (sizeof(T) == sizeof(double)) s = 1.0; else s = T{1.0, 0.0};
  } else {
    const double t = sqrt(aa * aa + bb * bb);
    c = aa / t;
    s = dscale(dconj(a), bb / (aa * t));
  }
  f.cs[j] = c;
  f.sn[j] = s;
  {
    const T p = Hj[j], q = Hj[j + 1];
    Hj[j] = c * p + dconj(s) * q;
    Hj[j + 1] = (-s) * p + c * q;
    const T gp = f.g[j], gq = f.g[j + 1];
    f.g[j] = c * gp + dconj(s) * gq;
    f.g[j + 1] = (-s) * gp + c * gq;
  }
  const int its = f.ints[1] + 1;
  f.ints[1] = its;
  f.ints[0] = j + 1;
  const double est = sqrt(dabs2(f.g[j + 1]));
  f.hist[its] = est / f.dbl[0];
  f.dbl[2] = hnext > 0 ? 1.0 / hnext : 0.0;
  if (est <= f.dbl[1] * f.dbl[0] || hnext <= 1e-14 * eta || its >= f.ints[2] || j + 1 >= m) *f.done = 1;
}

template <typename T>
__global__ void k_fgmres_col(FgmDev<T> f, int m, int j, const T *__restrict__ res1, const T *__restrict__ res2,
                             const T *__restrict__ res3) {
  if (*f.done) return;
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  fgmres_col_body(f, m, j, res1, res2, res3);
}

// The Givens column (thread 0 of CTA 0) and v_{j+1} = w / h_{j+1} (every CTA;
// h_{j+1} = ||w|| is res3[0], known to all) in one launch.
template <typename T>
__global__ void __launch_bounds__(256) k_fgmres_scale(FgmDev<T> f, int m, int j, const T *__restrict__ res1,
                                                      const T *__restrict__ res2, const T *__restrict__ res3, int64_t n,
                                                      const T *__restrict__ w, T *__restrict__ vnext) {
  pdl_launch();
  pdl_wait();
  if (*f.done) return;
  double hn2;
  if constexpr (sizeof(T) == sizeof(double)) hn2 = res3[0]; else hn2 = res3[0].x;
  const double hnext = sqrt(hn2 > 0 ? hn2 : 0.0);
  const double sc = hnext > 0 ? 1.0 / hnext : 0.0;
  if (blockIdx.x == 0) {
    // The Givens column on one thread, its inputs staged by the first warp (one
    // round trip for all; a thread walking them read them one L2 latency at a time)
    __shared__ T r1[GS_MAXC + 2], r2[GS_MAXC + 2], hcol[GS_MAXC + 2], sns[GS_MAXC];
    __shared__ double css[GS_MAXC];
    if (threadIdx.x < 32) {
      for (int i = threadIdx.x; i <= j + 1; i += 32) { r1[i] = res1[i]; r2[i] = res2[i]; }
      for (int i = threadIdx.x; i < j; i += 32) { css[i] = f.cs[i]; sns[i] = f.sn[i]; }
      __syncwarp();
      if (threadIdx.x == 0) {
        FgmDev<T> fs = f;
        fs.cs = css;
        fs.sn = sns;
        fs.H = hcol - (int64_t)j * (m + 1);                         // column j lands in hcol
        fgmres_col_body(fs, m, j, r1, r2, res3);
      }
      __syncwarp();
      T *Hj = f.H + (int64_t)j * (m + 1);
      for (int i = threadIdx.x; i <= j + 1; i += 32) Hj[i] = hcol[i];
      if (threadIdx.x == 0) { f.cs[j] = css[j]; f.sn[j] = sns[j]; }
    }
  }
  // CTA 0 only does the Givens column (a chain of small dependent loads); the other
  // CTAs scale, so the kernel ends at the later of the two instead of their sum
  if (gridDim.x > 1 && blockIdx.x == 0) return;
  const int64_t b0 = gridDim.x > 1 ? (int64_t)blockIdx.x - 1 : 0, nb = gridDim.x > 1 ? (int64_t)gridDim.x - 1 : 1;
  for (int64_t i = b0 * blockDim.x + threadIdx.x; i < n; i += nb * blockDim.x) vnext[i] = dscale(w[i], sc);
}

// ----------------------------------------------------------------- DCGS2 (c5', reading Q38)
// FGMRES with the lagged CGS2 of the oracle's fgmres_dcgs2: step j holds the not yet
// reorthogonalised, unnormalised u_j in column j of V (u_0 = r) and z_j = M(u_j).
// ONE dot pass   [c, a, nu, mu, eta^2] = [V_{0:j}^H u_j, V_{0:j}^H w, u_j^H u_j, u_j^H w, w^H w]
// (its last CTA completes column j - 1: alpha = sqrt(nu - |c|^2), Hraw[0:j, j-1] += c,
// Hraw[j, j-1] = alpha, the Givens rotation of that column, and h_j = (mu - c^H a) / alpha),
// then ONE update pass  v_j = (u_j - V c) / alpha (in place), u_{j+1} = w - V a - v_j h_j
// into column j + 1, ||u_{j+1}||^2 (its last CTA takes the stopping decision with the
// provisional H[j+1, j] = beta_j).  Two passes over the basis per iteration instead of
// CGS2's three, and no separate scaling pass.
template <typename T> __device__ inline double dre(T v);
template <> __device__ inline double dre<double>(double v) { return v; }
template <> __device__ inline double dre<cd>(cd v) { return v.x; }
template <typename T> __device__ inline T dfrom(double v);
template <> __device__ inline double dfrom<double>(double v) { return v; }
template <> __device__ inline cd dfrom<cd>(double v) { return cd{v, 0.0}; }

// dcs: [0] alpha, [1] h_j, [2] eta (as T), [3] ||u_{j+1}||^2 (reduced)
template <typename T>
struct DcgDev {
  FgmDev<T> f;
  T *Hraw;            // (m+1) x m column-major, unrotated
  T *dcs;             // 4 scalars
};

// Column completion of step j (warp 0 of the calling CTA; the other threads return).
// res = [c(j), a(j), nu, mu, eta^2] of the dot pass.  fin: the cycle's closing pass (no h_j).
template <typename T>
__device__ inline void dcgs_complete(DcgDev<T> d, int m, int j, int fin, const T *__restrict__ res) {
  __shared__ T hc[GS_MAXC + 2], sns[GS_MAXC];
  __shared__ double css[GS_MAXC];
  if (threadIdx.x >= 32) return;
  const int lane = threadIdx.x;
  FgmDev<T> &f = d.f;
  double cc = 0.0;
  T ca = dzero<T>();
  T *Hr = d.Hraw + (int64_t)(j > 0 ? j - 1 : 0) * (m + 1);
  for (int i = lane; i < j; i += 32) {
    const T c = res[i];
    cc += dabs2(c);
    if (!fin) ca += dconj(c) * res[j + i];
    const T h = Hr[i] + c;                                   // column j - 1 completed
    Hr[i] = h;
    hc[i] = h;
    if (i < j - 1) { css[i] = f.cs[i]; sns[i] = f.sn[i]; }
  }
  cc = warp_sum(cc);
  ca = warp_sum(ca);
  const double nu = dre(res[2 * j]);
  const double alpha = sqrt(fmax(nu - cc, 0.0));
  __syncwarp();
  if (lane == 0) {
    if (j == 0) {
      f.g[0] = dfrom<T>(alpha);                                // r = alpha v_0
    } else {
      const int jc = j - 1;
      Hr[j] = dfrom<T>(alpha);
      hc[j] = dfrom<T>(alpha);
      for (int i = 0; i < jc; ++i) {                           // previous rotations
        const T p = hc[i], q = hc[i + 1];
        hc[i] = css[i] * p + dconj(sns[i]) * q;
        hc[i + 1] = (-sns[i]) * p + css[i] * q;
      }
      const T a = hc[jc];
      const double aa = sqrt(dabs2(a)), bb = alpha;
      double c;
      T s;
      if (bb == 0.0) { c = 1.0; s = dzero<T>(); }
      else if (aa == 0.0) { c = 0.0; s = dfrom<T>(1.0); }
      else {
        const double t = sqrt(aa * aa + bb * bb);
        c = aa / t;
        s = dscale(dconj(a), bb / (aa * t));
      }
      f.cs[jc] = c;
      f.sn[jc] = s;
      const T p = hc[jc], q = hc[jc + 1];
      hc[jc] = c * p + dconj(s) * q;
      hc[jc + 1] = (-s) * p + c * q;
      const T gp = f.g[jc], gq = f.g[jc + 1];
      f.g[jc] = c * gp + dconj(s) * gq;
      f.g[jc + 1] = (-s) * gp + c * gq;
      const int its = f.ints[1] + 1;
      f.ints[1] = its;
      f.hist[its] = sqrt(dabs2(f.g[jc + 1])) / f.dbl[0];
    }
    if (!fin) {
      const T mu = res[2 * j + 1];
      d.dcs[0] = dfrom<T>(alpha);
      d.dcs[1] = dscale(mu - ca, 1.0 / alpha);                 // h_j = (mu - c^H a) / alpha
      d.dcs[2] = dfrom<T>(sqrt(fmax(dre(res[2 * j + 2]), 0.0)));
    }
  }
  __syncwarp();
  if (j > 0) {
    T *Hj = f.H + (int64_t)(j - 1) * (m + 1);
    for (int i = lane; i <= j; i += 32) Hj[i] = hc[i];
  }
}

// Stopping decision after the update pass of step j (warp 0): column j provisionally
// [a, h_j] with H[j+1, j] = beta_j; the estimate |g_j| beta_j / sqrt(|t_j|^2 + beta_j^2)
// after rotations 0..j-1 (the oracle's order), breakdown beta_j <= 1e-14 eta, maxit, m.
template <typename T>
__device__ inline void dcgs_check(DcgDev<T> d, int m, int j, const T *__restrict__ res) {
  __shared__ T sns[GS_MAXC];
  __shared__ double css[GS_MAXC];
  __shared__ T ta[GS_MAXC];
  if (threadIdx.x >= 32) return;
  const int lane = threadIdx.x;
  FgmDev<T> &f = d.f;
  T *Hr = d.Hraw + (int64_t)j * (m + 1);
  for (int i = lane; i < j; i += 32) {
    const T a = res[j + i];
    Hr[i] = a;
    ta[i] = a;
    css[i] = f.cs[i];
    sns[i] = f.sn[i];
  }
  __syncwarp();
  if (lane == 0) {
    const T hj = d.dcs[1];
    Hr[j] = hj;
    const double bj = sqrt(fmax(dre(d.dcs[3]), 0.0)), eta = dre(d.dcs[2]);
    // t_j after rotations 0..j-1 (only the last entry matters)
    T tj = j > 0 ? ta[0] : hj;
    for (int i = 0; i < j; ++i) {
      const T q = (i + 1 < j) ? ta[i + 1] : hj;
      tj = (-sns[i]) * tj + css[i] * q;                          // rotated entry i + 1
    }
    const double tt = sqrt(dabs2(tj) + bj * bj);
    const double gj = sqrt(dabs2(f.g[j]));
    const double est = tt > 0.0 ? gj * bj / tt : gj;
    f.ints[0] = j + 1;
    if (est <= f.dbl[1] * f.dbl[0] || bj <= 1e-14 * eta || f.ints[1] + 1 >= f.ints[2] || j + 1 >= m) *f.done = 1;
  }
}

// Dot pass of step j: grid (row blocks, ncg column groups); the columns are dealt to the
// groups in turn (group cg: c = cg + ncg (w + 8a), so the groups differ by at most one
// column); warp w owns the group's columns w + 8a, lanes the rows (TR per step, every load
// of a step in flight).  Column group 0's warp 0 also forms nu, mu, eta^2.  fuse: the last CTA
// completes column j - 1 (one GPU); else the caller all-reduces res and runs k_dgs_col.
// Last-CTA tail of the dot passes: the partials of all CTAs reduced in CTA order into
// res; fuse: column j - 1 completed by the same CTA.
template <typename T>
__device__ inline void dcgs_dot_tail(T *__restrict__ partial, int G, unsigned *ticket, T *__restrict__ res,
                                     DcgDev<T> d, int m, int ncols, int fin, int fuse) {
  __shared__ bool amlast;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) amlast = (atomicAdd(ticket, 1u) == gridDim.x * gridDim.y - 1);
  __syncthreads();
  if (!amlast) return;
  __threadfence();
  reduce_partials(partial, G, 2 * ncols + 3, res);
  if (threadIdx.x == 0) *ticket = 0;
  if (!fuse) return;
  __threadfence();
  __syncthreads();
  dcgs_complete(d, m, ncols, fin, res);
}

template <typename T, int NPW, int TR>
__global__ void __launch_bounds__(256, 2) k_dgs_dot(int64_t n, const T *__restrict__ V, int64_t ldv, int ncols,
                                                    const T *__restrict__ u, const T *__restrict__ w,
                                                    T *__restrict__ partial, unsigned *ticket, T *__restrict__ res,
                                                    const int *__restrict__ done, DcgDev<T> d, int m, int fin, int fuse) {
  pdl_launch();
  pdl_wait();
  if (done && *done) return;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nrb = gridDim.x, cg = blockIdx.y;
  T au[NPW], aw[NPW];
#pragma unroll
  for (int a = 0; a < NPW; ++a) { au[a] = dzero<T>(); aw[a] = dzero<T>(); }
  double nu = 0.0, et = 0.0;
  T mu = dzero<T>();
  const bool scal = (cg == 0 && warp == 0);
  const int ncg = gridDim.y;
  const int64_t nsteps = (n + 32 * TR - 1) / (32 * TR);
  for (int64_t step = blockIdx.x; step < nsteps; step += nrb) {
    const int64_t base = step * 32 * TR + lane;
    T vr[TR][NPW], ur[TR], wr[TR];
#pragma unroll
    for (int r = 0; r < TR; ++r) {
      const int64_t i = base + 32 * r;
      const bool ok = i < n;
      ur[r] = ok ? ld_nc(u + i) : dzero<T>();
      wr[r] = ok ? ld_nc(w + i) : dzero<T>();
#pragma unroll
      for (int a = 0; a < NPW; ++a) {
        const int c = cg + ncg * (warp + 8 * a);
        vr[r][a] = (ok && c < ncols) ? ld_nc(V + c * ldv + i) : dzero<T>();
      }
    }
#pragma unroll
    for (int r = 0; r < TR; ++r) {
#pragma unroll
      for (int a = 0; a < NPW; ++a) {
        const T cv = dconj(vr[r][a]);
        au[a] += cv * ur[r];
        aw[a] += cv * wr[r];
      }
      if (scal) {
        nu += dabs2(ur[r]);
        mu += dconj(ur[r]) * wr[r];
        et += dabs2(wr[r]);
      }
    }
  }
#pragma unroll
  for (int a = 0; a < NPW; ++a) {
    const int c = cg + ncg * (warp + 8 * a);
    const T su = warp_sum(au[a]), sw = warp_sum(aw[a]);
    if (lane == 0 && c < ncols) {
      partial[(int64_t)c * nrb + blockIdx.x] = su;
      partial[(int64_t)(ncols + c) * nrb + blockIdx.x] = sw;
    }
  }
  if (scal) {
    nu = warp_sum(nu);
    mu = warp_sum(mu);
    et = warp_sum(et);
    if (lane == 0) {
      partial[(int64_t)(2 * ncols) * nrb + blockIdx.x] = dfrom<T>(nu);
      partial[(int64_t)(2 * ncols + 1) * nrb + blockIdx.x] = mu;
      partial[(int64_t)(2 * ncols + 2) * nrb + blockIdx.x] = dfrom<T>(et);
    }
  }
  dcgs_dot_tail(partial, nrb, ticket, res, d, m, ncols, fin, fuse);
}

// Warp-tile form: lane i of a warp holds row 32 t + i of TU tiles with the NC columns of
// its column group (blockIdx.y: columns [NC y, NC y + NC)), u and w (no load shared between
// the warps, every value of TU tiles in flight); per-lane accumulators for the group's
// 2 NC results (group 0: + nu, mu, eta^2), summed over the lanes, the warps and the CTAs
// once at the end.  Groups > 0 re-read u and w (from L2 while the group waves overlap).
template <typename T, int NC, int TU>
__global__ void __launch_bounds__(256, (NC <= 8 && NC * TU * sizeof(T) <= 256) ? 2 : 1) k_dgs_dotw(int64_t n, const T *__restrict__ V, int64_t ldv, int ncols,
                                                  const T *__restrict__ u, const T *__restrict__ w,
                                                  T *__restrict__ partial, unsigned *ticket, T *__restrict__ res,
                                                  const int *__restrict__ done, DcgDev<T> d, int m, int fin, int fuse) {
  pdl_launch();
  pdl_wait();
  if (done && *done) return;
  __shared__ T red[8][2 * NC + 3];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  T au[NC], aw[NC];
#pragma unroll
  for (int c = 0; c < NC; ++c) { au[c] = dzero<T>(); aw[c] = dzero<T>(); }
  double nu = 0.0, et = 0.0;
  T mu = dzero<T>();
  const int64_t ntiles = (n + 31) / 32;
  const int c0 = blockIdx.y * NC, ng = min(NC, ncols - c0);
  const T *Vg = V + (int64_t)c0 * ldv;
  for (int64_t t0 = ((int64_t)blockIdx.x * 8 + warp) * TU; t0 < ntiles; t0 += (int64_t)gridDim.x * 8 * TU) {
    T v[TU][NC], ur[TU], wr[TU];
#pragma unroll
    for (int q = 0; q < TU; ++q) {
      const int64_t r = (t0 + q) * 32 + lane;
      const bool ok = r < n;
      ur[q] = ok ? ld_nc(u + r) : dzero<T>();
      wr[q] = ok ? ld_nc(w + r) : dzero<T>();
#pragma unroll
      for (int c = 0; c < NC; ++c) v[q][c] = (ok && c < ng) ? ld_nc(Vg + c * ldv + r) : dzero<T>();
    }
#pragma unroll
    for (int q = 0; q < TU; ++q) {
#pragma unroll
      for (int c = 0; c < NC; ++c) {
        const T cv = dconj(v[q][c]);
        au[c] += cv * ur[q];
        aw[c] += cv * wr[q];
      }
      nu += dabs2(ur[q]);
      mu += dconj(ur[q]) * wr[q];
      et += dabs2(wr[q]);
    }
  }
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    const T su = warp_sum(au[c]), sw = warp_sum(aw[c]);
    if (lane == 0) { red[warp][c] = su; red[warp][NC + c] = sw; }
  }
  nu = warp_sum(nu);
  mu = warp_sum(mu);
  et = warp_sum(et);
  if (lane == 0) {
    red[warp][2 * NC] = dfrom<T>(nu);
    red[warp][2 * NC + 1] = mu;
    red[warp][2 * NC + 2] = dfrom<T>(et);
  }
  __syncthreads();
  const int nl = 2 * ng + (blockIdx.y == 0 ? 3 : 0);            // this group's results
  for (int e = tid; e < nl; e += blockDim.x) {
    const int src = e < ng ? e : e < 2 * ng ? NC + (e - ng) : 2 * NC + (e - 2 * ng);
    const int q = e < ng ? c0 + e : e < 2 * ng ? ncols + c0 + (e - ng) : 2 * ncols + (e - 2 * ng);
    T t = dzero<T>();
#pragma unroll
    for (int k = 0; k < 8; ++k) t += red[k][src];
    partial[(int64_t)q * gridDim.x + blockIdx.x] = t;
  }
  dcgs_dot_tail(partial, (int)gridDim.x, ticket, res, d, m, ncols, fin, fuse);
}

template <typename T>
__global__ void k_dgs_col(DcgDev<T> d, int m, int j, int fin, const T *__restrict__ res, const int *__restrict__ done) {
  pdl_launch();
  pdl_wait();
  if (done && *done) return;
  dcgs_complete(d, m, j, fin, res);
}
template <typename T>
__global__ void k_dgs_check(DcgDev<T> d, int m, int j, const T *__restrict__ res, const int *__restrict__ done) {
  pdl_launch();
  pdl_wait();
  if (done && *done) return;
  dcgs_check(d, m, j, res);
}

// Update pass of step j: one thread per row (RPT rows, columns 8 at a time, all loads of a
// chunk in flight): s1 = V c, s2 = V a, v_j = (u_j - s1) / alpha (in place in column j),
// u_{j+1} = w - s2 - v_j h_j (column j + 1), ||u_{j+1}||^2 reduced in CTA order by the
// last CTA (fuse: which then takes the stopping decision).  pkdst: u_{j+1} also stored at
// its level-0 DOWN positions pkpos[i] (rows i < npk), the next apply's packed rhs.
template <typename T, int RPT, int CB = 8>
__global__ void __launch_bounds__(256) k_dgs_upd(int64_t n, T *V, int64_t ldv, int j, const T *__restrict__ w,
                                                 const T *__restrict__ res, T *__restrict__ partial, unsigned *ticket,
                                                 const int *__restrict__ done, DcgDev<T> d, int m, int fuse,
                                                 const int *__restrict__ pkpos, int64_t npk, T *__restrict__ pkdst) {
  pdl_launch();
  pdl_wait();
  if (done && *done) return;
  __shared__ T sc[GS_MAXC], sa[GS_MAXC];
  __shared__ double red[8];
  __shared__ bool amlast;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int i = tid; i < j; i += blockDim.x) { sc[i] = res[i]; sa[i] = res[j + i]; }
  const double ia = 1.0 / dre(d.dcs[0]);
  const T hj = d.dcs[1];
  __syncthreads();
  T *u = V + (int64_t)j * ldv, *un = V + (int64_t)(j + 1) * ldv;
  double nrm = 0.0;
  const int64_t chunk = 256 * RPT;
  for (int64_t b0 = (int64_t)blockIdx.x * chunk; b0 < n; b0 += (int64_t)gridDim.x * chunk) {
    T uu[RPT], ww[RPT], s1[RPT], s2[RPT];
#pragma unroll
    for (int k = 0; k < RPT; ++k) {
      const int64_t i = b0 + 256 * k + tid;
      const bool ok = i < n;
      uu[k] = ok ? u[i] : dzero<T>();
      ww[k] = ok ? ld_nc(w + i) : dzero<T>();
      s1[k] = dzero<T>();
      s2[k] = dzero<T>();
    }
    int c = 0;
    for (; c + CB <= j; c += CB) {
      T v[RPT][CB];
#pragma unroll
      for (int k = 0; k < RPT; ++k) {
        const int64_t i = b0 + 256 * k + tid;
#pragma unroll
        for (int q = 0; q < CB; ++q) v[k][q] = i < n ? ld_nc(V + (c + q) * ldv + i) : dzero<T>();
      }
#pragma unroll
      for (int k = 0; k < RPT; ++k)
#pragma unroll
        for (int q = 0; q < CB; ++q) {
          s1[k] += v[k][q] * sc[c + q];
          s2[k] += v[k][q] * sa[c + q];
        }
    }
    if (c < j) {                                                  // the last 1..CB-1 columns
      T v[RPT][CB];
#pragma unroll
      for (int k = 0; k < RPT; ++k) {
        const int64_t i = b0 + 256 * k + tid;
#pragma unroll
        for (int q = 0; q < CB; ++q) v[k][q] = (i < n && c + q < j) ? ld_nc(V + (c + q) * ldv + i) : dzero<T>();
      }
#pragma unroll
      for (int k = 0; k < RPT; ++k)
#pragma unroll
        for (int q = 0; q < CB; ++q)
          if (c + q < j) {
            s1[k] += v[k][q] * sc[c + q];
            s2[k] += v[k][q] * sa[c + q];
          }
    }
#pragma unroll
    for (int k = 0; k < RPT; ++k) {
      const int64_t i = b0 + 256 * k + tid;
      if (i < n) {
        const T vv = dscale(uu[k] - s1[k], ia);
        const T t = ww[k] - s2[k] - vv * hj;
        u[i] = vv;
        un[i] = t;
        nrm += dabs2(t);
        if (i < npk) {                                            // next apply's level-0 packed rhs
          const int p = pkpos[i];
          if (p >= 0) pkdst[p] = t;
        }
      }
    }
  }
  nrm = warp_sum(nrm);
  if (lane == 0) red[warp] = nrm;
  __syncthreads();
  if (tid == 0) {
    double s = 0.0;
#pragma unroll
    for (int q = 0; q < 8; ++q) s += red[q];
    partial[blockIdx.x] = dfrom<T>(s);
  }
  __threadfence();
  __syncthreads();
  if (tid == 0) amlast = (atomicAdd(ticket, 1u) == gridDim.x - 1);
  __syncthreads();
  if (!amlast) return;
  __threadfence();
  reduce_partials(partial, (int)gridDim.x, 1, d.dcs + 3);
  if (tid == 0) *ticket = 0;
  if (!fuse) return;
  __threadfence();
  __syncthreads();
  dcgs_check(d, m, j, res);
}

// ----------------------------------------------------------------- NEXT-1 root GMRES helpers
// Start of the root-level inner GMRES (Alg. 2 line 6): beta = ||z2||
// from the norm pass, the inner state reset, the inner done flag copied from the
// outer one (an outer FGMRES that has finished skips the whole inner solve).
template <typename T>
__global__ void k_root_start(FgmDev<T> f, int m, const T *__restrict__ res, const int *__restrict__ outer_done,
                             int *__restrict__ skip) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  double b2;
  if constexpr (sizeof(T) == sizeof(double)) b2 = res[0]; else b2 = res[0].x;
  const double beta = sqrt(b2 > 0 ? b2 : 0.0);
  const int od = outer_done ? *outer_done : 0;
  *skip = od;
  f.dbl[0] = beta > 0 ? beta : 1.0;     // "bnorm" of the inner residual history
  f.dbl[1] = 0.0;                       // no tolerance test: a fixed number of steps (or breakdown)
  f.dbl[4] = beta > 0 ? 1.0 / beta : 0.0;
  f.ints[0] = 0;
  f.ints[1] = 0;
  f.ints[2] = 1 << 30;
  for (int i = 0; i <= m; ++i) f.g[i] = dzero<T>();
  if constexpr (sizeof(T) == sizeof(double)) f.g[0] = beta; else f.g[0] = T{beta, 0.0};
  *f.done = (od || beta == 0.0) ? 1 : 0;
}
// y = H[0:jend, 0:jend]^{-1} g (upper triangular after the rotations), zero beyond jend
template <typename T>
__global__ void k_root_solve(FgmDev<T> f, int m, const int *__restrict__ skip, T *__restrict__ y) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  if (*skip) return;
  const int jend = f.ints[0];
  for (int i = m - 1; i >= 0; --i) {
    if (i >= jend) { y[i] = dzero<T>(); continue; }
    T acc = f.g[i];
    for (int c = i + 1; c < jend; ++c) acc -= f.H[(int64_t)c * (m + 1) + i] * y[c];
    y[i] = acc / f.H[(int64_t)i * (m + 1) + i];
  }
}

// ----------------------------------------------------------------- utilities
// y = x * scale[0] (scale may be a device scalar of 1/β); done-guarded
template <typename T>
__global__ void k_scale(int64_t n, const T *x, T *y, const double *scale, const int *done) {
  if (done && *done) return;
  const double sc = *scale;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    y[i] = dscale(x[i], sc);
}

// x += Z[:, 0:ncols] y
template <typename T>
__global__ void k_xupdate(int64_t n, const T *__restrict__ Z, int64_t ldz, int ncols, const T *__restrict__ y, T *x) {
  __shared__ T sy[GS_MAXC];
  for (int c = threadIdx.x; c < ncols; c += blockDim.x) sy[c] = y[c];
  __syncthreads();
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    T acc = x[i];
    for (int c = 0; c < ncols; ++c) acc += ld_nc(Z + c * ldz + i) * sy[c];
    x[i] = acc;
  }
}

// out[:, c] = V[:, 0:m] Y[:, c], c < kc (thick-restart basis rotation)
template <typename T>
__global__ void k_gemm_tall(int64_t n, const T *__restrict__ V, int64_t ldv, int m, const T *__restrict__ Y, int kc,
                            T *__restrict__ out, int64_t ldo) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    for (int c0 = 0; c0 < kc; c0 += 8) {
      T acc[8];
#pragma unroll
      for (int a = 0; a < 8; ++a) acc[a] = dzero<T>();
      for (int j = 0; j < m; ++j) {
        const T v = V[j * ldv + i];
#pragma unroll
        for (int a = 0; a < 8; ++a)
          if (c0 + a < kc) acc[a] += v * Y[(int64_t)(c0 + a) * m + j];
      }
#pragma unroll
      for (int a = 0; a < 8; ++a)
        if (c0 + a < kc) out[(c0 + a) * ldo + i] = acc[a];
    }
  }
}

// natural <-> permuted: local[i] = natural[perm[i]]  /  natural[perm[i]] = local[i]
template <typename T>
__global__ void k_perm(int64_t n, const int64_t *__restrict__ perm, const T *__restrict__ in, T *__restrict__ out,
                       int inverse) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    if (inverse) out[perm[i]] = in[i]; else out[i] = in[perm[i]];
  }
}

template <typename T>
__global__ void k_fill(int64_t n, T *x, T v) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) x[i] = v;
}

}  // namespace gemslr
