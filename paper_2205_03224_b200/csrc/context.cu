// GeMSLR solve path on one B200: device plan, orchestration and the C-ABI
// (include/gemslr.h).  arXiv 2205.03224, /root/reference/PAPER.md = "P".
//
//   spmv            K1                                   (Note N P:L58-61)
//   apply_precond   Alg. 2 single pass: down sweep (K4, K6+K7, K8) -> bottom
//                   block-Jacobi (K9) -> up sweep (K5)
//   solve           FGMRES(m) with CGS2 (K10-K12), device-side Givens, host
//                   least squares per cycle
//   setup           host plan (hostplan.cpp) + bottom-up thick-restart Arnoldi
//                   on Ĝ_l with the same kernels
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <memory>
#include <random>
#include <set>
#include <type_traits>
#include <string>
#include <dlfcn.h>
#include <sys/stat.h>
#include <type_traits>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "../../include/gemslr.h"
#include "kernels.cuh"
#include "plan.hpp"

namespace gemslr {

// SMs of the current device (cudaDevAttrMultiProcessorCount; sizes the grids and
// the cooperative k_ewx launch, so a partitioned GPU — MIG, MPS limits — still works)
// E_l's columns: local (or U-packed) positions below kHaloE, halo entries at
// kHaloE + index (the E kernels take nloc = kHaloE); packed positions may exceed
// the local length, so the split point cannot be n.
static constexpr int32_t kHaloE = 1 << 30;

static int num_sm() {
  static int cache[64] = {0};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) dev = 0;
  if (!cache[dev]) {
    int v = 0;
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v <= 0) v = 148;
    cache[dev] = v;
  }
  return cache[dev];
}
long long *g_tri_dbg = nullptr;   // debug: per-chunk clock64 trace of block 0 (gemslr_debug_trace)
int g_tri_dbg_level = 0;          // level whose down launch is traced
static_assert(PIPE_SB == PIPE_SB_DEV && PIPE_NW == PIPE_NW_DEV, "pipeline constants");

#define CK(x)                                                                          \
  do {                                                                                 \
    cudaError_t e_ = (x);                                                              \
    if (e_ != cudaSuccess) throw Error{GEMSLR_ERR_CUDA, std::string("CUDA: ") + #x + ": " + cudaGetErrorString(e_)}; \
  } while (0)

// host scalar <-> device scalar
template <typename T> struct Dev;
template <> struct Dev<double> { using type = double; };
template <> struct Dev<zc> { using type = cd; };

// ----------------------------------------------------------------- device memory
struct Allocator {
  void *(*alloc_fn)(size_t, void *) = nullptr;
  void (*free_fn)(void *, void *) = nullptr;
  void *user = nullptr;
  void *alloc(size_t bytes) {
    if (bytes == 0) bytes = 16;
    void *p = nullptr;
    if (alloc_fn) p = alloc_fn(bytes, user);
    else if (cudaMalloc(&p, bytes) != cudaSuccess) p = nullptr;
    if (!p) throw Error{GEMSLR_ERR_OOM, "device allocation of " + std::to_string(bytes) + " bytes failed"};
    return p;
  }
  void release(void *p) {
    if (!p) return;
    if (free_fn) free_fn(p, user); else cudaFree(p);
  }
};

struct Pool {                                   // owns every device allocation of a context
  Allocator *A = nullptr;
  std::vector<void *> ptrs;
  size_t bytes = 0;
  template <typename U>
  U *get(size_t count) {
    U *p = static_cast<U *>(A->alloc(count * sizeof(U)));
    ptrs.push_back(p);
    bytes += count * sizeof(U);
    return p;
  }
  template <typename U, typename V>
  U *upload(const std::vector<V> &h, cudaStream_t s) {
    static_assert(sizeof(U) == sizeof(V), "layout");
    U *p = get<U>(std::max<size_t>(h.size(), 1));
    if (!h.empty()) CK(cudaMemcpyAsync(p, h.data(), h.size() * sizeof(U), cudaMemcpyHostToDevice, s));
    return p;
  }
  void clear() {
    for (void *p : ptrs) A->release(p);
    ptrs.clear();
    bytes = 0;
  }
};

// ----------------------------------------------------------------- profiling
enum KernelClass { KC_SPMV = 0, KC_TRI_DOWN, KC_TRI_UP, KC_TRI_LAST, KC_EW, KC_WAXPY, KC_GS, KC_FGM, KC_UTIL, KC_PACK, KC_COUNT };
static const char *kKernelName[KC_COUNT] = {"spmv", "trisolve_down", "trisolve_up", "trisolve_last", "ew",
                                            "waxpy", "gs", "fgmres_col", "util", "pack_rhs"};

struct Profiler {
  bool on = false;
  struct Rec { int kc, sub; cudaEvent_t a, b; };
  std::vector<Rec> pending;
  std::vector<cudaEvent_t> freelist;
  double ms[KC_COUNT] = {0};
  long long count[KC_COUNT] = {0};
  double sub_ms[KC_COUNT][4] = {{0}};         // per level (trisolve classes)
  cudaEvent_t ev() {
    if (!freelist.empty()) { cudaEvent_t e = freelist.back(); freelist.pop_back(); return e; }
    cudaEvent_t e;
    cudaEventCreate(&e);
    return e;
  }
  void flush() {
    for (auto &r : pending) {
      cudaEventSynchronize(r.b);
      float t = 0;
      cudaEventElapsedTime(&t, r.a, r.b);
      ms[r.kc] += t;
      count[r.kc] += 1;
      sub_ms[r.kc][std::min(r.sub, 3)] += t;
      freelist.push_back(r.a);
      freelist.push_back(r.b);
    }
    pending.clear();
  }
  void reset() {
    flush();
    for (int i = 0; i < KC_COUNT; ++i) {
      ms[i] = 0;
      count[i] = 0;
      for (int q = 0; q < 4; ++q) sub_ms[i][q] = 0;
    }
  }
  ~Profiler() {
    for (auto &r : pending) { cudaEventDestroy(r.a); cudaEventDestroy(r.b); }
    for (auto e : freelist) cudaEventDestroy(e);
  }
};

struct Timed {                                  // RAII event pair around one launch
  Profiler &P;
  cudaStream_t s;
  int kc, sub;
  cudaEvent_t a = nullptr;
  Timed(Profiler &p, cudaStream_t st, int k, int sb = 0) : P(p), s(st), kc(k), sub(sb) {
    if (P.on) { a = P.ev(); cudaEventRecord(a, s); }
  }
  ~Timed() {
    if (P.on) {
      cudaEvent_t b = P.ev();
      cudaEventRecord(b, s);
      P.pending.push_back({kc, sub, a, b});
      if (P.pending.size() > 4096) P.flush();
    }
  }
};

// ----------------------------------------------------------------- NCCL (dlopen)
// The library loads NCCL at run time (the torch wheel's libnccl.so.2, or the
// one already loaded in the process) so it links against no NCCL at build time.
struct Comm {
  void *lib = nullptr;
  void *comm = nullptr;
  bool owned = false;
  int nranks = 1, rank = 0;
  bool force = false;          // one-rank NCCL communicator driving the distributed path (tests, bench)
  typedef int (*fn_uid)(void *);
  typedef int (*fn_init)(void **, int, const void *, int);   // id passed by value: see init()
  typedef int (*fn_destroy)(void *);
  typedef int (*fn_allreduce)(const void *, void *, size_t, int, int, void *, cudaStream_t);
  typedef int (*fn_p2p)(const void *, size_t, int, int, void *, cudaStream_t);
  typedef int (*fn_recv)(void *, size_t, int, int, void *, cudaStream_t);
  typedef int (*fn_group)();
  typedef const char *(*fn_err)(int);
  typedef int (*fn_count)(void *, int *);
  fn_allreduce allreduce_ = nullptr;
  fn_p2p send_ = nullptr;
  fn_recv recv_ = nullptr;
  fn_group gstart_ = nullptr, gend_ = nullptr;
  fn_err errstr_ = nullptr;
  fn_destroy destroy_ = nullptr;
  long long allreduces = 0, exchanges = 0;

  static void *open_lib(const char *path) {
    void *h = nullptr;
    if (path && *path) h = dlopen(path, RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) throw Error{GEMSLR_ERR_NCCL, "cannot load libnccl.so.2"};
    return h;
  }
  template <typename F> F sym(const char *name) {
    F f = reinterpret_cast<F>(dlsym(lib, name));
    if (!f) throw Error{GEMSLR_ERR_NCCL, std::string("NCCL symbol missing: ") + name};
    return f;
  }
  void bind() {
    allreduce_ = sym<fn_allreduce>("ncclAllReduce");
    send_ = sym<fn_p2p>("ncclSend");
    recv_ = sym<fn_recv>("ncclRecv");
    gstart_ = sym<fn_group>("ncclGroupStart");
    gend_ = sym<fn_group>("ncclGroupEnd");
    errstr_ = sym<fn_err>("ncclGetErrorString");
    destroy_ = sym<fn_destroy>("ncclCommDestroy");
  }
  void check(int rc, const char *what) {
    if (rc != 0) throw Error{GEMSLR_ERR_NCCL, std::string("NCCL ") + what + ": " + (errstr_ ? errstr_(rc) : "error")};
  }
  void borrow(void *c, const char *path) {
    lib = open_lib(path);
    bind();
    comm = c;
    int n = 1, r = 0;
    check(sym<fn_count>("ncclCommCount")(c, &n), "CommCount");
    check(sym<fn_count>("ncclCommUserRank")(c, &r), "CommUserRank");
    nranks = n;
    rank = r;
  }
  void init(const char *path, int n, int r, const void *id128) {
    lib = open_lib(path);
    bind();
    // ncclCommInitRank(ncclComm_t*, int, ncclUniqueId (128 bytes by value), int)
    struct Id { char b[128]; } id;
    std::memcpy(id.b, id128, 128);
    typedef int (*fn_init_v)(void **, int, Id, int);
    check(sym<fn_init_v>("ncclCommInitRank")(&comm, n, id, r), "CommInitRank");
    owned = true;
    nranks = n;
    rank = r;
  }
  // host-staged backend (gemslr_create_hostcomm): the caller's callbacks move
  // host buffers (e.g. torch.distributed over gloo); device data is staged
  // through pinned host memory after a stream synchronisation
  gemslr_allreduce_fn h_allreduce = nullptr;
  gemslr_sendrecv_fn h_sendrecv = nullptr;
  void *h_user = nullptr;
  double *hbuf = nullptr;
  size_t hcap = 0;
  double *host(size_t ndouble) {
    if (ndouble > hcap) {
      if (hbuf) cudaFreeHost(hbuf);
      hcap = std::max<size_t>(ndouble, 1 << 16);
      if (cudaMallocHost(&hbuf, hcap * sizeof(double)) != cudaSuccess) throw Error{GEMSLR_ERR_OOM, "pinned staging"};
    }
    return hbuf;
  }
  bool hostmode() const { return h_allreduce != nullptr; }
  // sum over ranks in place; count in doubles (complex = 2 doubles each)
  void allreduce(void *buf, size_t ndouble, cudaStream_t s) {
    if ((nranks == 1 && !force) || ndouble == 0) return;
    if (hostmode()) {
      double *h = host(ndouble);
      if (cudaMemcpyAsync(h, buf, ndouble * 8, cudaMemcpyDeviceToHost, s) != cudaSuccess || cudaStreamSynchronize(s) != cudaSuccess)
        throw Error{GEMSLR_ERR_CUDA, "host-staged all-reduce copy"};
      if (h_allreduce(h_user, h, ndouble) != 0) throw Error{GEMSLR_ERR_NCCL, "host all-reduce callback failed"};
      if (cudaMemcpyAsync(buf, h, ndouble * 8, cudaMemcpyHostToDevice, s) != cudaSuccess || cudaStreamSynchronize(s) != cudaSuccess)
        throw Error{GEMSLR_ERR_CUDA, "host-staged all-reduce copy"};
    } else {
      check(allreduce_(buf, buf, ndouble, 8 /*ncclFloat64*/, 0 /*ncclSum*/, comm, s), "AllReduce");
    }
    allreduces++;
  }
  ~Comm() {
    if (owned && comm && destroy_) destroy_(comm);
    if (hbuf) cudaFreeHost(hbuf);
  }
};

// ----------------------------------------------------------------- device plan
template <typename D>
struct StageDev {
  int nblk = 0, cps = 1;
  int64_t rows = 0, row0 = 0;
  const int64_t *blk = nullptr;
  TriDev<D> L{}, U{};
  int depthL = 0, depthU = 0;
  bool pipe = false;       // TMA-pipelined kernel (k_tri_pipe) instead of the level kernel
  PipeDev<D> P{};
  bool reg = false;        // register-prefetched kernel (k_tri_reg), preferred when available
  int reg_w = 0;           // record width W (4, 8, 10, 12 or 16)
  int reg_nw = 0;          // consumer warps of k_tri_reg (reg_nw_for)
  int reg_q = 1;           // split form: CTAs (a cluster) per block
  int reg_la = 0;          // look-ahead new columns of the records (0 or REG_LA)
  RegDev<D> Rg{};
  int64_t reg_bytes = 0;   // record bytes of both sweeps
  const int *lrow = nullptr;       // per packed L position: the row (-1 padding), DOWN gather
  D *rhs_up = nullptr;             // UP right-hand sides (zero except the F_l rows)
  const int *urow = nullptr;       // per packed U position: the row (-1 padding)
  D *xU = nullptr;                 // UP: the level's x in U-packed order (k_pack_f), updated in place by k_tri_reg
  const int *fpos = nullptr, *frow = nullptr;
  int64_t nf = -1;                 // rows with F_l entries (-1: not set up, use k_pack_rhs)
  int64_t lslices = 0, uslices = 0;
  // several right-hand sides (NEXT-4): per-column packed buffers, mcap columns
  D *mL = nullptr, *mU = nullptr, *mUp = nullptr;
  int mcap = 0;
  int64_t nchunks = 0, far = 0, nearc = 0;
  int64_t nnz = 0;         // real stored nonzeros (L + U incl. diagonal)
  int64_t padded = 0;      // stored entries incl. padding
  // tail form (plan.hpp TailPack, DESIGN 6b) of the one-column apply's DOWN / UP
  bool tail = false;
  RegDev<D> TD{}, TU{};
  int td_w = 0, td_nw = 0, td_la = 0, tu_w = 0, tu_nw = 0, tu_la = 0;
  size_t td_smem = 0, tu_smem = 0;
  const int *tlrow = nullptr;      // per DOWN L position: the row (-1 padding)
  int64_t tnL = 0;                 // DOWN L positions
  const int *tpos = nullptr;       // row -> its DOWN L position (-1: none), rows < ntpos (DCGS2 pre-packing)
  int64_t ntpos = 0;
  D *trhsL = nullptr;              // DOWN right-hand sides ([L_hh | L_t|h] order)
  D *tT = nullptr;                 // t = L^-1 b1 (Ucat order)
  D *tu = nullptr;                 // u = L_tt^-1 (F_l y2)_tail (U_tt order)
  D *tz = nullptr;                 // z1 on the tail (U_tt order; E_l reads it)
  D *trhsU = nullptr;              // (F_l y2)_tail in L_tt order (zero off the F_l rows)
  const int *tfpos = nullptr;      // L_tt position of every row with F_l entries
  const int *tfrow = nullptr;      // those rows (F_l row index)
  int64_t tnf = 0;
  int depth_tail[6] = {0, 0, 0, 0, 0, 0};   // L_hh, L_t|h, U_tt, L_tt, U_tt, U_h|t
  int64_t tail_rows = 0, tail_bytes = 0;
  int64_t tail_nnz[5] = {0, 0, 0, 0, 0};   // stored entries of L_hh, L_t|h, U_tt (no diagonal), U_h|t, L_tt
  D *rhs_packed_buf() const { return tail ? trhsL : const_cast<D *>(Rg.rhsL); }
};

template <typename D>
struct CsrDev {
  int64_t n = 0, nnz = 0;
  const int64_t *ptr = nullptr;
  const int32_t *col = nullptr;
  const D *val = nullptr;
};

template <typename D>
struct LevelDev {
  int64_t o0 = 0, o1 = 0, s = 0;
  StageDev<D> st;
  CsrDev<D> E, F;
  // one GPU, register trisolve: E_l's columns as U-packed positions of the level's
  // stage, so E_l z1 reads z1 from the U-packed copy the DOWN trisolve writes (xpm)
  const int32_t *Ecol_p = nullptr;
  const int32_t *esidx_p = nullptr;  // several ranks: hE's send indices as U-packed positions
  // one GPU: k_ewx also writes the first npk rows of r_J (the next stage's rows)
  // at their packed L positions pkpos in that stage's right-hand-side buffer
  int64_t npk = 0;
  const int *pkpos = nullptr;
  int k = 0;
  D *W = nullptr;          // s x k column-major, ld = ldw
  int64_t ldw = 0;
  D *G = nullptr;          // k x k
  std::vector<typename std::conditional<std::is_same<D, double>::value, double, zc>::type> Wh, Rh, Gh;  // host copies
  int cycles = 0;
};

struct Ctx;

template <typename D>
struct HaloDev {                  // device side of a HaloPlan
  std::vector<int32_t> peer;
  std::vector<int64_t> soff, roff;
  const int *sidx = nullptr;
  D *sbuf = nullptr, *rbuf = nullptr;
  int64_t nsend = 0, nrecv = 0;
};

template <typename T>
struct Engine {
  using D = typename Dev<T>::type;
  Ctx *ctx = nullptr;
  HostPlan<T> plan;
  int64_t n = 0, nnzA = 0;
  // SpMV (SELL-32 of Â)
  int64_t nslices = 0, sell_padded = 0, sell_wmax = 0;
  // long / uneven rows: warp-per-row CSR SpMV (k_spmv_wpr) instead of SELL-32
  bool use_wpr = false;
  const int64_t *csr_ptr = nullptr;
  const int32_t *csr_col = nullptr;
  const D *csr_val = nullptr;
  const int64_t *sell_off = nullptr;
  const int32_t *sell_col = nullptr;
  const D *sell_val = nullptr;
  std::vector<LevelDev<D>> lev;
  StageDev<D> last;
  const int64_t *perm_d = nullptr;   // natural (original) row of every local row
  // distributed SpMV: the SELL slices without / with halo columns, so the halo
  // exchange (on comm_stream) overlaps the interior slices (north_star; Note N P:L58-63)
  const int *sl_in = nullptr, *sl_bd = nullptr;
  int64_t n_in = 0, n_bd = -1;
  cudaStream_t comm_stream = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  bool dist = false;                 // distributed path: several ranks, or a forced one-rank NCCL communicator
  HaloDev<D> hA;
  std::vector<HaloDev<D>> hE, hF;
  D *rl_full = nullptr, *yl_full = nullptr;   // replicated last separator (nranks > 1)
  const int *last_idx_d = nullptr;
  int64_t nglob = 0, o_last = 0;
  // workspace
  D *r = nullptr, *tmp = nullptr, *tvec = nullptr, *partial = nullptr, *res = nullptr;
  unsigned *tickets = nullptr;
  int *ewflag = nullptr;             // k_ewx generation counter (device-side)
  unsigned *gtickets = nullptr;      // k_ewg grid-barrier ticket counters, one per level (apply_from)
  size_t partial_cap = 0;
  // Krylov workspace (lazy)
  int kry_m = -1;
  int64_t ldv = 0;
  D *V = nullptr, *Z = nullptr, *w = nullptr;
  D *H = nullptr, *g = nullptr, *sn = nullptr, *ydev = nullptr;
  double *cs = nullptr, *dbl = nullptr, *hist = nullptr;
  int *ints = nullptr, *done = nullptr;
  D *Hraw = nullptr, *dcs = nullptr;   // DCGS2: unrotated Hessenberg, [alpha, h_j, eta, beta_j^2]
  int hist_cap = 0;
  D *xb = nullptr, *bb = nullptr;   // host-path staging
  int *hflags = nullptr;             // pinned: done flag of every iteration of a cycle (async D2H)
  int hflags_cap = 0;
  char *hstage = nullptr;            // pinned: the cycle-end state (counters, history, H, g)
  size_t hstage_cap = 0;
  std::vector<cudaGraphExec_t> graphs;   // FGMRES iteration j captured once (one GPU)
  int graph_m = -1;
  const D *graph_V = nullptr;
  const double *graph_hist = nullptr;  // captured k_fgmres_scale nodes write hist: a new buffer needs new graphs
  int graph_orth = -1;
  cudaStream_t cap_stream = nullptr;
  ~Engine() {
    if (ev_fork) cudaEventDestroy(ev_fork);
    if (ev_join) cudaEventDestroy(ev_join);
    if (comm_stream) cudaStreamDestroy(comm_stream);
    if (hflags) cudaFreeHost(hflags);
    if (hstage) cudaFreeHost(hstage);
    for (auto &ge : graphs) if (ge) cudaGraphExecDestroy(ge);
    if (cap_stream) cudaStreamDestroy(cap_stream);
  }
  double setup_host_s = 0, setup_dev_s = 0, arnoldi_s = 0;

  void upload(cudaStream_t s);
  void exchange(HaloDev<D> &h, const D *src, const int *doneflag, cudaStream_t comm_st = nullptr,
                const int *sidx = nullptr);
  void allreduce(D *buf, size_t count);
  void apply_from(int l0, const D *in, D *out, const int *doneflag, bool in_packed = false);
  bool prepack_ok() const;
  // several right-hand sides (NEXT-4, one GPU): column-major n x nr blocks, leading dimension ld
  D *rM = nullptr, *tmpM = nullptr;
  int64_t multi_cap = 0;                                            // nr * ld of rM / tmpM
  bool multi_ok() const;
  void ensure_multi(int nr, int64_t ld);
  void apply_multi(const D *in, D *out, int64_t ld, int nr);
  void spmv_multi(const D *x, D *y, int64_t ld, int nr);
  void ew_column(LevelDev<D> &d, int l, const D *src, const D *z, D *dst, const int *doneflag = nullptr);
  // NEXT-1: root-level inner GMRES on Ŝ_0 (one GPU)
  int root_its = 0;
  D *Vr = nullptr, *Zr = nullptr, *wr = nullptr, *ur = nullptr, *zerov = nullptr, *Hr = nullptr, *gr = nullptr,
    *snr = nullptr, *yr = nullptr, *rres = nullptr;
  double *csr = nullptr, *dblr = nullptr, *histr = nullptr;
  int *intsr = nullptr, *doner = nullptr, *skipr = nullptr;
  int64_t ldr = 0;
  void root_gmres(const D *bJ, D *xJ, const int *doneflag);
  void spmv(const D *x, D *y, int mode, const D *b, const int *doneflag);
  void ghat(int l, D *bufA, D *bufB);
  void build_lowrank(const gemslr_params &prm, unsigned long long seed);
  int solve(const D *b, D *x, double rtol, int m, int maxit, int *its, double *hist, int hcap, int *hlen, double *frel);
  void ensure_krylov(int m, int maxit);
  void gs_pass(const D *Vb, int64_t ldvv, int64_t nn, int ncols, D *wv, int upd, int dot, const D *h_in, D *resv, int ticket, const int *doneflag);
  double norm(const D *x, int64_t nn, int ticket);
  void dgs_step(int j, int m, int fin, const int *doneflag);
  void export_bundle(const std::string &dir) const;
  std::string stats_json() const;
};

struct Ctx {
  int device = -1;
  int orth = 0;                      // FGMRES orthogonalisation: 0 CGS2 (c5), 1 DCGS2 (c5', reading Q38)
  cudaStream_t stream = nullptr;
  Comm comm;
  Allocator alloc;
  Pool pool;
  Profiler prof;
  std::string err;
  int dtype = -1;
  bool ready = false;
  bool host_only = false;
  int coord_dim = 0;
  std::vector<double> coords;
  const double *coords_src = nullptr;
  gemslr_params params{};
  std::unique_ptr<Engine<double>> ed;
  std::unique_ptr<Engine<zc>> ez;
};

// ----------------------------------------------------------------- upload
// Consumer warps of k_tri_reg for a stage.  A warp's record loads are issued
// right after its slice and waited for at its next one, NW slices later, i.e.
// NW / K levels later with K slices per level: stages with many slices per
// level (the level-0 subdomains) need more warps to cover the L2 latency, stages
// with 1-2 slices per level pay for the wider barriers.  K = all slices / all
// levels of the stage's blocks.  GEMSLR_REG_NW overrides (experiments).
template <typename D, typename T>
static int reg_nw_for(const RegPack<T> &R) {
  static const int env = getenv("GEMSLR_REG_NW") ? atoi(getenv("GEMSLR_REG_NW")) : 0;
  const int nb = (int)(R.binfo.size() / REG_BINFO_INTS);
  int64_t sl = 0, lv = 0;
  for (int b = 0; b < nb; ++b) {
    const int32_t *bi = &R.binfo[(size_t)b * REG_BINFO_INTS];
    sl += bi[1] + bi[4] + (R.nsweep == 3 ? bi[7] : 0);
    lv += bi[2] + bi[5] + (R.nsweep == 3 ? bi[8] : 0);
  }
  const double K = lv > 0 ? (double)sl / (double)lv : 1.0;
  if (sizeof(D) == 8) {
    if (env == 15 || env == 23) return env;
    // tail form of the deep stages (one CTA streams a whole level-0 block's records, the
    // per-SM bytes in flight bound it): 31 warps, one buffer each, 64 registers (spill-free
    // up to W = 12).  C5 level 0: DOWN / UP 235 / 253 -> 211 / 235 us per apply vs 23 warps.
    if (R.nsweep == 3 && K >= 2.5 && R.W <= 12 && env != 23) return 31;
    // split chunks (C5 level 0 at Q = 4: K = 2.8): 23 warps measured 4 % faster than 15
    return K >= (R.Q > 1 ? 2.5 : 3.0) ? 23 : 15;
  }
  if (env == 7 || env == 15) return env;
  return 15;                                                       // complex: 15 warps, one buffer (C4: every level)
}

template <typename D, typename T>
static StageDev<D> upload_stage(Pool &P, cudaStream_t s, const Stage<T> &S, int cps_override, int tri_kernel) {
  StageDev<D> d;
  d.nblk = (int)S.blk.size() - 1;
  d.rows = S.blk.empty() ? 0 : S.blk.back() - S.blk.front();
  d.row0 = S.blk.empty() ? 0 : S.blk.front();
  d.blk = P.upload<int64_t>(S.blk, s);
  auto up = [&](const TriPack<T> &p) {
    TriDev<D> t;
    t.blk_lev = P.upload<int32_t>(p.blk_lev, s);
    t.lev_slice = P.upload<int32_t>(p.lev_slice, s);
    t.slice_off = P.upload<int64_t>(p.slice_off, s);
    t.slice_row = P.upload<int32_t>(p.slice_row, s);
    t.col = P.upload<int32_t>(p.col, s);
    t.val = P.upload<D>(p.val, s);
    t.diag = p.diag.empty() ? nullptr : P.upload<D>(p.diag, s);
    return t;
  };
  d.L = up(S.Lp);
  d.U = up(S.Up);
  d.depthL = S.Lp.max_depth;
  d.depthU = S.Up.max_depth;
  if (S.pipe.ok && cps_override <= 0 && tri_kernel != 2 && d.nblk > 0 && pipe_smem_bytes<D>(S.pipe.ring) <= 232448) {
    static_assert(sizeof(ChunkDesc) == sizeof(ChunkDev), "chunk descriptor layout");
    d.pipe = true;
    d.P.blob = P.upload<unsigned char>(S.pipe.blob, s);
    d.P.chunks = P.upload<ChunkDev>(S.pipe.chunks, s);
    d.P.blk_chunk = P.upload<int>(S.pipe.blk_chunk, s);
    d.P.blk_nl = P.upload<int>(S.pipe.blk_nl, s);
    d.P.lpos = P.upload<int>(S.pipe.lpos, s);
    d.P.row0 = S.blk.front();
    d.P.rhsL = P.get<D>(std::max<int64_t>(S.pipe.lslices * 32, 1));
    d.P.rhsU = P.get<D>(std::max<int64_t>(S.pipe.uslices * 32, 1));
    d.P.ring = S.pipe.ring;
    d.nchunks = (int64_t)S.pipe.chunks.size();
    d.far = S.pipe.far;
    d.nearc = S.pipe.near;
  }
  if (S.reg.ok && cps_override <= 0 && tri_kernel == 0 && d.nblk > 0 &&
      reg_smem_bytes<D>(S.reg.ring, S.reg.max_block_slices, S.reg.imp_L + S.reg.imp_U, S.reg.plev_L + S.reg.plev_U,
                        S.reg.Q > 1) <= 232448 - 1024) {
    static_assert(REG_BINFO == REG_BINFO_INTS && REG_LA == REG_LA_DEV, "record layout");
    d.reg = true;
    d.reg_w = S.reg.W;
    d.reg_nw = reg_nw_for<D>(S.reg);
    d.Rg.data = P.upload<unsigned char>(S.reg.data, s);
    d.Rg.slev = P.upload<unsigned short>(S.reg.slev, s);
    d.Rg.max_slices = S.reg.max_block_slices;
    d.Rg.rec_bytes = (long long)S.reg.rec_bytes;
    d.Rg.binfo = P.upload<int>(S.reg.binfo, s);
    d.Rg.lev_off = P.upload<int>(S.reg.lev_off, s);
    d.Rg.rhsL = P.get<D>(std::max<int64_t>(S.reg.lslices * 32, 1));
    d.lrow = P.upload<int>(S.Lp.slice_row, s);
    d.lslices = S.reg.lslices;
    d.uslices = S.reg.uslices;
    d.rhs_up = P.get<D>(std::max<int64_t>(S.reg.lslices * 32, 1));
    CK(cudaMemsetAsync(d.rhs_up, 0, std::max<int64_t>(S.reg.lslices * 32, 1) * sizeof(D), s));
    d.Rg.mid = P.get<D>(std::max<int64_t>(S.reg.uslices * 32, 1));
    d.urow = P.upload<int>(S.Up.slice_row, s);
    d.xU = P.get<D>(std::max<int64_t>(S.reg.uslices * 32, 1));
    d.Rg.ring = S.reg.ring;
    d.reg_q = S.reg.Q;
    d.reg_la = S.reg.la;
    d.Rg.Q = S.reg.Q;
    d.Rg.imp_L = S.reg.imp_L;
    d.Rg.imp_U = S.reg.imp_U;
    d.Rg.plev_L = S.reg.plev_L;
    d.Rg.plev_U = S.reg.plev_U;
    d.Rg.sneed = S.reg.Q > 1 ? P.upload<unsigned short>(S.reg.sneed, s) : nullptr;
    d.Rg.xexp = S.reg.Q > 1 ? P.upload<unsigned short>(S.reg.xexp, s) : nullptr;
    d.Rg.xp = S.reg.xmode ? 1 : 0;
    d.reg_bytes = (int64_t)S.reg.data.size();
    if (!d.pipe) d.P.lpos = P.upload<int>(S.reg.lpos, s);
  }
  // tail form: only next to the one-CTA / split register kernel (the same record format)
  const bool no_tail = getenv("GEMSLR_TAIL") && atoi(getenv("GEMSLR_TAIL")) != 1;   // 0 off, 2 order only
  if (S.tail.ok && !no_tail && d.nblk > 0 && cps_override <= 0 && tri_kernel == 0) {
    const TailPack<T> &TP = S.tail;
    auto mk = [&](const RegPack<T> &R, RegDev<D> &G, int &w, int &nw, int &la, size_t &smem) {
      G = RegDev<D>{};
      G.data = P.upload<unsigned char>(R.data, s);
      G.slev = P.upload<unsigned short>(R.slev, s);
      G.max_slices = R.max_block_slices;
      G.rec_bytes = (long long)R.rec_bytes;
      G.binfo = P.upload<int>(R.binfo, s);
      G.ring = R.ring;
      G.Q = 1;
      G.imp_L = R.imp_L;
      G.xp = 1;
      w = R.W;
      nw = reg_nw_for<D>(R);
      la = R.la;
      smem = reg_smem_bytes<D>(R.ring, R.max_block_slices, R.imp_L, 0, false);
      return smem <= 232448 - 1024;
    };
    bool ok = mk(TP.D, d.TD, d.td_w, d.td_nw, d.td_la, d.td_smem);
    ok = mk(TP.U, d.TU, d.tu_w, d.tu_nw, d.tu_la, d.tu_smem) && ok;
    if (ok) {
      d.tail = true;
      d.tnL = (int64_t)TP.lrow.size();
      d.tlrow = P.upload<int>(TP.lrow, s);
      {
        int64_t mx = -1;
        for (int r : TP.lrow) mx = std::max<int64_t>(mx, r);
        std::vector<int> inv((size_t)(mx + 1), -1);
        for (size_t q = 0; q < TP.lrow.size(); ++q)
          if (TP.lrow[q] >= 0) inv[(size_t)TP.lrow[q]] = (int)q;
        d.ntpos = mx + 1;
        if (d.ntpos > 0) d.tpos = P.upload<int>(inv, s);
      }
      const int64_t nU = (int64_t)TP.Utt.slice_row.size() + (int64_t)TP.Uht.slice_row.size();
      d.trhsL = P.get<D>(std::max<int64_t>(d.tnL, 1));
      CK(cudaMemsetAsync(d.trhsL, 0, std::max<int64_t>(d.tnL, 1) * sizeof(D), s));
      d.tT = P.get<D>(std::max<int64_t>(nU, 1));
      d.tu = P.get<D>(std::max<int64_t>(TP.nUtt, 1));
      d.tz = P.get<D>(std::max<int64_t>(TP.nUtt, 1));
      const int64_t nLtt = std::max<int64_t>((int64_t)TP.Ltt.slice_row.size(), 1);
      d.trhsU = P.get<D>(nLtt);
      CK(cudaMemsetAsync(d.trhsU, 0, nLtt * sizeof(D), s));
      // DOWN: L_hh, L_t|h -> t (Ucat), U_tt -> z1 (U_tt order)
      RegDev<D> &A = d.TD;
      A.ra[0] = d.trhsL; A.roff[0] = 0; A.st[0] = d.tT; A.stm[0] = 0; A.upper[0] = 0;
      A.ra[1] = d.trhsL; A.roff[1] = TP.nLhh; A.st[1] = d.tT; A.stm[1] = 0; A.upper[1] = 0;
      A.ra[2] = d.tT; A.roff[2] = 0; A.st[2] = d.tz; A.stm[2] = 1; A.upper[2] = 1;
      // UP: L_tt -> u, U_tt on t - u -> x, U_h|t on t -> x (x set per launch)
      RegDev<D> &B = d.TU;
      B.ra[0] = d.trhsU; B.roff[0] = 0; B.st[0] = d.tu; B.stm[0] = 0; B.upper[0] = 0;
      B.ra[1] = d.tT; B.rb[1] = d.tu; B.roff[1] = 0; B.stm[1] = 0; B.upper[1] = 1;
      B.ra[2] = d.tT; B.roff[2] = TP.nUtt; B.stm[2] = 0; B.upper[2] = 1;
      d.depth_tail[0] = TP.Lhh.max_depth;
      d.depth_tail[1] = TP.Lth.max_depth;
      d.depth_tail[2] = TP.Utt.max_depth;
      d.depth_tail[3] = TP.Ltt.max_depth;
      d.depth_tail[4] = TP.Utt.max_depth;
      d.depth_tail[5] = TP.Uht.max_depth;
      d.tail_rows = TP.tail_rows;
      d.tail_nnz[0] = TP.Lhh.nnz_real;
      d.tail_nnz[1] = TP.Lth.nnz_real;
      d.tail_nnz[2] = TP.Utt.nnz_real;
      d.tail_nnz[3] = TP.Uht.nnz_real;
      d.tail_nnz[4] = TP.Ltt.nnz_real;
      d.tail_bytes = (int64_t)(TP.D.data.size() + TP.U.data.size());
    }
  }
  if (S.reg.Q > 1 && !d.reg)                                       // chunks are not independent blocks
    throw Error{GEMSLR_ERR_INVALID_ARG, "split triangular solves need the register-prefetched kernel"};
  d.nnz = S.Lp.nnz_real + S.Up.nnz_real + (int64_t)d.rows;
  d.padded = (int64_t)S.Lp.val.size() + (int64_t)S.Up.val.size() + (int64_t)S.Up.diag.size();
  // CTAs per block: enough to cover the average rows of one level with 8-warp CTAs,
  // bounded by the SMs available per block and the portable cluster size.
  int cps = 1;
  if (cps_override > 0) cps = cps_override;
  else if (d.nblk > 0) {
    const double depth = std::max(1, std::max(d.depthL, d.depthU));
    const double rows_per_level = (double)d.rows / d.nblk / depth;
    int want = (int)std::ceil(rows_per_level / 256.0);
    int avail = std::max(1, num_sm() / d.nblk);
    cps = std::min(std::min(want, avail), 8);
    int p2 = 1;
    while (p2 * 2 <= cps) p2 *= 2;
    cps = std::max(1, p2);
  }
  d.cps = std::min(cps, 8);
  return d;
}

template <typename D, typename T>
static CsrDev<D> upload_csr(Pool &P, cudaStream_t s, const Csr<T> &A) {
  CsrDev<D> d;
  d.n = A.n;
  d.nnz = A.nnz();
  d.ptr = P.upload<int64_t>(A.ptr, s);
  d.col = P.upload<int32_t>(A.col, s);
  d.val = P.upload<D>(A.val, s);
  return d;
}

template <typename D>
static HaloDev<D> upload_halo(Pool &P, cudaStream_t s, const HaloPlan &h) {
  HaloDev<D> d;
  d.peer = h.peer;
  d.soff = h.soff;
  d.roff = h.roff;
  d.nsend = h.nsend();
  d.nrecv = h.nrecv();
  d.sidx = P.upload<int>(h.sidx, s);
  d.sbuf = P.get<D>(std::max<int64_t>(d.nsend, 1));
  d.rbuf = P.get<D>(std::max<int64_t>(d.nrecv, 1));
  return d;
}

template <typename T>
void Engine<T>::upload(cudaStream_t s) {
  Pool &P = ctx->pool;
  const auto &A = plan.Aloc;                   // owned rows of Â, local / halo columns
  n = plan.nloc;
  nglob = plan.st.n;
  o_last = plan.st.o[plan.st.L];
  nnzA = A.nnz();
  // SELL-32 of the owned rows
  nslices = (n + 31) / 32;
  std::vector<int64_t> off(nslices + 1, 0);
  for (int64_t sl = 0; sl < nslices; ++sl) {
    int64_t w = 0;
    for (int64_t row = sl * 32; row < std::min(n, sl * 32 + 32); ++row) w = std::max(w, A.ptr[row + 1] - A.ptr[row]);
    off[sl + 1] = off[sl] + 32 * w;
  }
  sell_padded = off[nslices];
  for (int64_t sl = 0; sl < nslices; ++sl) sell_wmax = std::max<int64_t>(sell_wmax, (off[sl + 1] - off[sl]) / 32);
  std::vector<int32_t> col(sell_padded, -1);
  std::vector<T> val(sell_padded, T(0));
  for (int64_t row = 0; row < n; ++row) {
    const int64_t sl = row / 32, lane = row % 32;
    for (int64_t p = A.ptr[row], e = 0; p < A.ptr[row + 1]; ++p, ++e) {
      col[off[sl] + 32 * e + lane] = A.col[p];
      val[off[sl] + 32 * e + lane] = A.val[p];
    }
  }
  sell_off = P.upload<int64_t>(off, s);
  sell_col = P.upload<int32_t>(col, s);
  sell_val = P.upload<D>(val, s);
  {
    // SELL pads every lane of a slice to the slice's longest row: rows of 32+
    // entries on average, or more than half the stored entries padding, go to the
    // warp-per-row kernel (GEMSLR_SPMV=sell / wpr forces one)
    const double avg = n > 0 ? (double)nnzA / (double)n : 0.0;
    use_wpr = avg >= 32.0 || (double)sell_padded > 2.0 * (double)std::max<int64_t>(nnzA, 1);
    if (const char *e = getenv("GEMSLR_SPMV")) use_wpr = std::string(e) == "wpr";
    if (use_wpr) {
      csr_ptr = P.upload<int64_t>(A.ptr, s);
      csr_col = P.upload<int32_t>(A.col, s);
      csr_val = P.upload<D>(A.val, s);
    }
  }
  if (dist) {
    std::vector<int32_t> in, bd;
    for (int64_t sl = 0; sl < nslices; ++sl) {
      bool halo = false;
      for (int64_t e = off[sl]; e < off[sl + 1] && !halo; ++e) halo = col[e] >= n;
      (halo ? bd : in).push_back((int32_t)sl);
    }
    sl_in = P.upload<int32_t>(in, s);
    sl_bd = P.upload<int32_t>(bd, s);
    n_in = (int64_t)in.size();
    n_bd = (int64_t)bd.size();
  }
  std::vector<int64_t> nat(n);
  for (int64_t i = 0; i < n; ++i) nat[i] = plan.st.perm[plan.gpos[i]];
  perm_d = P.upload<int64_t>(nat, s);
  const int L = plan.st.L;
  lev.resize(L);
  hE.resize(L);
  hF.resize(L);
  for (int l = 0; l < L; ++l) {
    LevelDev<D> &d = lev[l];
    d.o0 = plan.lo[l];
    d.o1 = plan.lo[l + 1];
    d.s = n - d.o1;
    d.st = upload_stage<D>(P, s, plan.stage[l], ctx->params.cluster_ctas, ctx->params.tri_kernel);
    d.E = upload_csr<D>(P, s, plan.E[l]);
    {                                                              // E's halo columns at kHaloE + index
      std::vector<int32_t> ec(plan.E[l].col);
      for (auto &c : ec)
        if (c >= n) c = kHaloE + (int32_t)(c - n);
      d.E.col = P.upload<int32_t>(ec, s);
    }
    d.F = upload_csr<D>(P, s, plan.F[l]);
    if (d.st.reg) {                                                // sparse UP pack: the rows with F_l entries
      const auto &Fh = plan.F[l];
      const Stage<T> &S = plan.stage[l];
      const int64_t R0 = S.blk.empty() ? 0 : S.blk.front();
      std::vector<int32_t> fpos, frow;
      bool ok = true;
      for (int64_t i = 0; i < Fh.n && ok; ++i) {
        if (Fh.ptr[i + 1] == Fh.ptr[i]) continue;
        const int64_t row = d.o0 + i - R0;
        if (row < 0 || row >= (int64_t)S.reg.lpos.size() || S.reg.lpos[row] < 0) ok = false;
        else {
          fpos.push_back(S.reg.lpos[row]);
          frow.push_back((int32_t)i);
        }
      }
      if (ok) {
        d.st.fpos = P.upload<int>(fpos, s);
        d.st.frow = P.upload<int>(frow, s);
        d.st.nf = (int64_t)fpos.size();
      }
      if (d.st.xU && d.st.nf >= 0) {                 // the UP then reads z1 from xU (k_pack_f path)
        const auto &Eh = plan.E[l];
        std::vector<int32_t> upos(S.reg.lpos.size(), -1);
        for (size_t q = 0; q < S.Up.slice_row.size(); ++q) {
          const int64_t row = (int64_t)S.Up.slice_row[q] - R0;
          if (S.Up.slice_row[q] >= 0 && row >= 0 && row < (int64_t)upos.size()) upos[row] = (int32_t)q;
        }
        auto packed = [&](int64_t lrow_) -> int32_t {               // local row -> U-packed position, -1 if none
          const int64_t row = lrow_ - R0;
          return (row < 0 || row >= (int64_t)upos.size()) ? -1 : upos[row];
        };
        std::vector<int32_t> ecp(Eh.col.size());
        bool eok = true;
        for (size_t q = 0; q < Eh.col.size() && eok; ++q) {
          if (Eh.col[q] >= n) { ecp[q] = kHaloE + (int32_t)(Eh.col[q] - n); continue; }   // halo: as in E.col
          ecp[q] = packed(Eh.col[q]);
          eok = ecp[q] >= 0;
        }
        // several ranks: the z1 values this rank sends for the others' E_l are read
        // from the same U-packed copy
        std::vector<int32_t> sp(plan.hE[l].sidx.size());
        for (size_t q = 0; q < sp.size() && eok; ++q) {
          sp[q] = packed(plan.hE[l].sidx[q]);
          eok = sp[q] >= 0;
        }
        if (eok && !ecp.empty()) {
          d.Ecol_p = P.upload<int32_t>(ecp, s);
          d.esidx_p = P.upload<int32_t>(sp, s);
        }
      }
    }
    if (d.st.tail) {                                               // tail form: positions in its packs
      const auto &Fh = plan.F[l], &Eh = plan.E[l];
      const Stage<T> &S = plan.stage[l];
      const TailPack<T> &TP = S.tail;
      const int64_t R0 = S.blk.empty() ? 0 : S.blk.front();
      auto at = [&](const std::vector<int32_t> &pos, int64_t lrow_) -> int32_t {
        const int64_t row = lrow_ - R0;
        return (row < 0 || row >= (int64_t)pos.size()) ? -1 : pos[row];
      };
      bool ok = true;
      std::vector<int32_t> fpos, frow;
      for (int64_t i = 0; i < Fh.n && ok; ++i) {
        if (Fh.ptr[i + 1] == Fh.ptr[i]) continue;
        fpos.push_back(at(TP.lttpos, d.o0 + i));
        frow.push_back((int32_t)i);
        ok = fpos.back() >= 0;
      }
      std::vector<int32_t> ecp(Eh.col.size()), sp(plan.hE[l].sidx.size());
      for (size_t q = 0; q < Eh.col.size() && ok; ++q) {
        if (Eh.col[q] >= n) { ecp[q] = kHaloE + (int32_t)(Eh.col[q] - n); continue; }
        ecp[q] = at(TP.uttpos, Eh.col[q]);
        ok = ecp[q] >= 0;
      }
      for (size_t q = 0; q < sp.size() && ok; ++q) {
        sp[q] = at(TP.uttpos, plan.hE[l].sidx[q]);
        ok = sp[q] >= 0;
      }
      if (ok) {
        d.st.tfpos = P.upload<int>(fpos, s);
        d.st.tfrow = P.upload<int>(frow, s);
        d.st.tnf = (int64_t)fpos.size();
        d.Ecol_p = P.upload<int32_t>(ecp, s);
        d.esidx_p = P.upload<int32_t>(sp, s);
      } else {
        d.st.tail = false;
      }
    }
    hE[l] = upload_halo<D>(P, s, plan.hE[l]);
    hF[l] = upload_halo<D>(P, s, plan.hF[l]);
  }
  hA = upload_halo<D>(P, s, plan.hA);
  last = upload_stage<D>(P, s, plan.last_stage, ctx->params.cluster_ctas, ctx->params.tri_kernel);
  {                                                                // packed next-stage right-hand sides from k_ewx / k_waxpy
    for (int l = 0; l < L; ++l) {
      if (dist && l + 1 == L) continue;                            // several ranks: C_last is gathered and replicated
      LevelDev<D> &d = lev[l];
      const Stage<T> &NS = (l + 1 < L) ? plan.stage[l + 1] : plan.last_stage;
      StageDev<D> &nd = (l + 1 < L) ? lev[l + 1].st : last;
      if (!nd.reg || NS.blk.empty() || d.s <= 0) continue;
      const int64_t R0n = NS.blk.front();
      const int64_t npk = ((l + 1 < L) ? plan.lo[l + 2] : n) - d.o1;
      if (npk <= 0 || npk > d.s) continue;
      std::vector<int32_t> pos(npk);
      bool ok = true;
      const std::vector<int32_t> &lp = nd.tail ? NS.tail.lcat : NS.reg.lpos;   // the stage's DOWN L positions
      for (int64_t i = 0; i < npk && ok; ++i) {
        // (the last stage numbers its rows from o_L: make_stage's relative bounds)
        const int64_t row = d.o1 + i - (l + 1 < L ? R0n : plan.lo[L] + R0n);
        if (row < 0 || row >= (int64_t)lp.size() || lp[row] < 0) ok = false;
        else pos[i] = lp[row];
      }
      if (!ok) continue;
      d.pkpos = P.upload<int>(pos, s);
      d.npk = npk;
      if (nd.tail) CK(cudaMemsetAsync(nd.trhsL, 0, std::max<int64_t>(nd.tnL, 1) * sizeof(D), s));
      else CK(cudaMemsetAsync(const_cast<D *>(nd.Rg.rhsL), 0, std::max<int64_t>(nd.lslices * 32, 1) * sizeof(D), s));
    }
  }
  if (dist) {
    rl_full = P.get<D>(plan.slast + 1);
    yl_full = P.get<D>(plan.slast + 1);
    last_idx_d = P.upload<int>(plan.last_idx, s);
  }
  r = P.get<D>(n + 1);
  tmp = P.get<D>(n + 1);
  tvec = P.get<D>(64 * 8);
  partial_cap = (size_t)num_sm() * 8 * (GS_MAXC + 2);
  partial = P.get<D>(partial_cap);
  res = P.get<D>(4 * (GS_MAXC + 2));
  tickets = P.get<unsigned>(16);
  ewflag = P.get<int>(1);
  CK(cudaMemsetAsync(ewflag, 0, sizeof(int), s));
  gtickets = P.get<unsigned>(std::max(L, 1));
  CK(cudaMemsetAsync(gtickets, 0, std::max(L, 1) * sizeof(unsigned), s));
  CK(cudaMemsetAsync(tickets, 0, 16 * sizeof(unsigned), s));
  CK(cudaMemsetAsync(r, 0, (n + 1) * sizeof(D), s));
  CK(cudaMemsetAsync(tmp, 0, (n + 1) * sizeof(D), s));
}

// Neighbour exchange: pack src[sidx] and send/receive with every
// peer in one NCCL group on the solver stream.  No-op on one GPU.
template <typename T>
void Engine<T>::exchange(HaloDev<D> &h, const D *src, const int *doneflag, cudaStream_t comm_st, const int *sidx) {
  if (h.peer.empty()) return;
  Comm &C = ctx->comm;
  const int w = (int)(sizeof(D) / sizeof(double));
  if (h.nsend > 0) {
    const int grid = (int)std::min<int64_t>((h.nsend + 255) / 256, 4 * num_sm());
    k_gather_idx<D><<<grid, 256, 0, ctx->stream>>>(h.nsend, sidx ? sidx : h.sidx, src, h.sbuf, doneflag);
    CK(cudaGetLastError());
  }
  if (comm_st) {                                                   // the caller forked comm_st after the pack
    CK(cudaEventRecord(ev_fork, ctx->stream));
    CK(cudaStreamWaitEvent(comm_st, ev_fork, 0));
  } else {
    comm_st = ctx->stream;
  }
  if (C.hostmode()) {
    const size_t ns = (size_t)h.nsend * w, nr = (size_t)h.nrecv * w;
    double *hs = C.host(ns + nr);
    double *hr = hs + ns;
    CK(cudaMemcpyAsync(hs, h.sbuf, ns * 8, cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    std::vector<const double *> sp;
    std::vector<double *> rp;
    std::vector<size_t> sc, rc;
    for (size_t i = 0; i < h.peer.size(); ++i) {
      sp.push_back(hs + h.soff[i] * w);
      sc.push_back((size_t)(h.soff[i + 1] - h.soff[i]) * w);
      rp.push_back(hr + h.roff[i] * w);
      rc.push_back((size_t)(h.roff[i + 1] - h.roff[i]) * w);
    }
    if (C.h_sendrecv(C.h_user, (int)h.peer.size(), h.peer.data(), sp.data(), sc.data(), rp.data(), rc.data()) != 0)
      throw Error{GEMSLR_ERR_NCCL, "host send/recv callback failed"};
    CK(cudaMemcpyAsync(h.rbuf, hr, nr * 8, cudaMemcpyHostToDevice, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
  } else {
    C.check(C.gstart_(), "GroupStart");
    for (size_t i = 0; i < h.peer.size(); ++i) {
      const int64_t ns = h.soff[i + 1] - h.soff[i], nr = h.roff[i + 1] - h.roff[i];
      if (ns > 0) C.check(C.send_(h.sbuf + h.soff[i], (size_t)ns * w, 8, h.peer[i], C.comm, comm_st), "Send");
      if (nr > 0) C.check(C.recv_(h.rbuf + h.roff[i], (size_t)nr * w, 8, h.peer[i], C.comm, comm_st), "Recv");
    }
    C.check(C.gend_(), "GroupEnd");
  }
  C.exchanges++;
}

template <typename T>
void Engine<T>::allreduce(D *buf, size_t count) {
  ctx->comm.allreduce(buf, count * (sizeof(D) / sizeof(double)), ctx->stream);
}

// ----------------------------------------------------------------- launches
// Launch with programmatic stream serialization (PDL): the kernel's CTAs may be
// scheduled while its predecessor runs; the kernel's pdl_wait() orders its
// reads after the predecessor (kernels.cuh).  GEMSLR_NO_PDL=1 launches normally.
template <typename... KA, typename... A>
static void launch_pdl(void (*kern)(KA...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, A &&...args) {
  static const bool on = getenv("GEMSLR_NO_PDL") == nullptr;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = on ? 1 : 0;
  CK(cudaLaunchKernelEx(&cfg, kern, std::forward<A>(args)...));
}

// The same with a thread-block cluster of `csize` CTAs along x (the split form of
// k_tri_reg: one cluster per subdomain block).
template <typename... KA, typename... A>
static void launch_pdl_cluster(void (*kern)(KA...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, int csize,
                               A &&...args) {
  static const bool on = getenv("GEMSLR_NO_PDL") == nullptr;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = (unsigned)csize;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = on ? 2 : 1;
  CK(cudaLaunchKernelEx(&cfg, kern, std::forward<A>(args)...));
}

static int grid_for(int64_t units, int per_sm) {
  int64_t g = std::min<int64_t>(units, (int64_t)num_sm() * per_sm);
  return (int)std::max<int64_t>(g, 1);
}

// The k_ew / k_ewx instance for k low-rank columns: NACC = ceil(k / 8) accumulators
// per warp, rounded up to 1, 2, 3, 4, 6 or 8 (k <= 64).
template <typename F>
static void with_nacc(int k, F &&f) {
  if (k > EW_MAXK) throw Error{GEMSLR_ERR_INVALID_ARG, "low rank k > 64 in the E/W coupling"};
  if (k <= 8) f(std::integral_constant<int, 1>{});
  else if (k <= 16) f(std::integral_constant<int, 2>{});
  else if (k <= 24) f(std::integral_constant<int, 3>{});
  else if (k <= 32) f(std::integral_constant<int, 4>{});
  else if (k <= 48) f(std::integral_constant<int, 6>{});
  else f(std::integral_constant<int, 8>{});
}

// K6 + K7 (rows J_l: dst = src - E z ; this rank's part of s = W^H dst into sout)
template <typename D>
static void launch_ew(cudaStream_t st, int64_t s, int64_t rowbase, const int64_t *Eptr, const int32_t *Ecol,
                      const D *Eval, const D *z, const D *zh, int64_t nloc, const D *src, D *dst, const D *W,
                      int64_t ldw, int k, D *partial, unsigned *ticket, D *sout, const int *done) {
  const int grid = grid_for((std::max<int64_t>(s, 1) + 255) / 256, 4);
  with_nacc(k, [&](auto nc) {
    k_ew<D, decltype(nc)::value><<<grid, 256, 0, st>>>(s, rowbase, Eptr, Ecol, Eval, z, zh, nloc, src, dst, W, ldw, k,
                                                        partial, ticket, sout, done);
  });
  CK(cudaGetLastError());
}

// K6 + K7 + K8 in one cooperative launch (k_ewx): every CTA must be co-resident,
// so the grid is capped by the occupancy of the instance on this device.
template <typename D>
static void launch_ewx(cudaStream_t st, int64_t s, int64_t rowbase, const int64_t *Eptr, const int32_t *Ecol,
                       const D *Eval, const D *z, const D *zh, int64_t nloc, const D *src, D *dst, const D *W,
                       int64_t ldw, int k, const D *G, D *partial, unsigned *ticket, D *sout, int *flag,
                       const int *done, int64_t npk, const int *pkpos, D *pk, unsigned *gticket = nullptr) {
  // small interface (<= 8 CTAs of one row per thread, k <= 32): one cluster (k_ewc)
  static const int small_max = getenv("GEMSLR_EWC_MAX") ? atoi(getenv("GEMSLR_EWC_MAX")) : 2048;
  if (s <= std::min(small_max, 8 * 256) && k <= 32) {
    const int C = (int)std::max<int64_t>(1, (s + 255) / 256);
    with_nacc(k, [&](auto nc) {
      constexpr int NA = decltype(nc)::value;
      if constexpr (NA <= 4)
        launch_pdl_cluster(k_ewc<D, NA>, dim3(C), dim3(256), 0, st, C, s, rowbase, Eptr, Ecol, Eval, z, zh, nloc, src, dst,
                           W, ldw, k, G, done, npk, pkpos, pk);
    });
    return;
  }
  // large interface with a grid that fits the SMs: the PDL / grid-barrier form (k_ewg)
  static const bool no_ewg = getenv("GEMSLR_NO_EWG") != nullptr;
  if (gticket && k <= 32 && !no_ewg) {
    bool launched = false;
    with_nacc(k, [&](auto nc) {
      constexpr int NA = decltype(nc)::value;
      if constexpr (NA <= 4) {
        auto kern = k_ewg<D, NA>;
        static int cap[64] = {0};                                  // co-resident CTAs per device
        int dev = 0;
        cudaGetDevice(&dev);
        dev = (dev >= 0 && dev < 64) ? dev : 0;
        if (cap[dev] == 0) {
          int per = 0;
          CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kern, 256, 0));
          cap[dev] = std::max(1, per) * num_sm();
        }
        const int64_t grid = (std::max<int64_t>(s, 1) + 255) / 256;
        if (grid <= cap[dev]) {
          launch_pdl(kern, dim3((unsigned)grid), dim3(256), 0, st, s, rowbase, Eptr, Ecol, Eval, z, zh, nloc, src, dst, W,
                     ldw, k, G, partial, gticket, done, npk, pkpos, pk);
          launched = true;
        }
      }
    });
    if (launched) return;
  }
  with_nacc(k, [&](auto nc) {
    auto kern = k_ewx<D, decltype(nc)::value>;
    static int max_ctas[64] = {0};                                  // per device
    int dev = 0;
    cudaGetDevice(&dev);
    dev = (dev >= 0 && dev < 64) ? dev : 0;
    if (max_ctas[dev] == 0) {
      int per = 0;
      CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kern, 256, 0));
      max_ctas[dev] = std::max(1, per) * num_sm();
    }
    const int grid = (int)std::min<int64_t>((std::max<int64_t>(s, 1) + 255) / 256, max_ctas[dev]);
    void *args[] = {&s, &rowbase, &Eptr, &Ecol, &Eval, &z, &zh, &nloc, &src, &dst, &W, &ldw, &k, &G, &partial,
                    &ticket, &sout, &flag, &done, &npk, &pkpos, &pk};
    CK(cudaLaunchCooperativeKernel((const void *)kern, dim3(grid), dim3(256), args, 0, st));
  });
}

// F_l product arguments of an UP launch: y_J from the local vector, the halo
// and (nranks > 1) the replicated last separator.
template <typename D>
struct FArgs {
  const CsrDev<D> *F = nullptr;
  int64_t Fbase = 0, nloc = 0, nh = 0;
  const D *yh = nullptr, *yl = nullptr;
};

// Tail form of a level's DOWN / UP (plan.hpp TailPack, DESIGN 6b), one right-hand side:
// DOWN packs b1 ([L_hh | L_t|h] order; or k_ewx already did), then one k_tri_reg<TAIL>
// launch: t -> S.tT, z1 on the tail -> S.tz.  UP packs (F_l y2)_tail (k_pack_f), then
// one launch: y1 -> x[I_l].
template <typename D>
static void launch_tail(Ctx *ctx, const StageDev<D> &S, bool down, const D *rhs, D *x, const FArgs<D> &fa,
                        const int *doneflag, int kc, int lvl, bool rhs_packed) {
  if (S.nblk <= 0 || S.rows == 0) return;
  {
    {
      // (profiler: a pack is timed and counted only when a kernel is launched)
      if (down && !rhs_packed) {
        const Timed tt(ctx->prof, ctx->stream, KC_PACK);
        launch_pdl(k_pack_gather<D>, dim3(grid_for((S.tnL + 255) / 256, 4), 1), dim3(256), 0, ctx->stream, S.tnL,
                   S.tlrow, rhs, S.trhsL, doneflag, (int64_t)0, (int64_t)0);
      } else if (!down && S.tnf > 0) {
        const Timed tt(ctx->prof, ctx->stream, KC_PACK);
        const CsrDev<D> *F = fa.F;
        launch_pdl(k_pack_f<D>, dim3(grid_for((S.tnf + 255) / 256, 4), 1), dim3(256), 0, ctx->stream, (int64_t)S.tnf,
                   S.tfpos, S.tfrow, F->ptr, F->col, F->val, (const D *)x, (int64_t)fa.nloc, fa.yh, (int64_t)fa.nh, fa.yl,
                   S.trhsU, doneflag, (int64_t)0, (int64_t)0, (int64_t)0, (const int *)nullptr, (D *)nullptr);
      }
    }
    RegDev<D> Rg = down ? S.TD : S.TU;
    if (!down) Rg.st[1] = Rg.st[2] = x;
    const int w = down ? S.td_w : S.tu_w, nw = down ? S.td_nw : S.tu_nw, la = down ? S.td_la : S.tu_la;
    const size_t smem = down ? S.td_smem : S.tu_smem;
    Timed t(ctx->prof, ctx->stream, kc, lvl);
    auto go = [&](auto kern) {
      static std::set<const void *> attr;
      if (attr.insert((const void *)kern).second)
        CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 232448 - 1024));
      launch_pdl(kern, dim3(S.nblk, 1), dim3(32 * nw), smem, ctx->stream, Rg, (int)TRI_DOWN, x, (D *)nullptr, doneflag);
    };
    auto by_w = [&](auto nwc, auto nbc, auto lac) {
      constexpr int NW = decltype(nwc)::value, NB = decltype(nbc)::value, LA = decltype(lac)::value;
      switch (w) {
        case 4: go(k_tri_reg<D, 4, NW, NB, false, LA, true>); break;
        case 8: go(k_tri_reg<D, 8, NW, NB, false, LA, true>); break;
        case 10: go(k_tri_reg<D, 10, NW, NB, false, LA, true>); break;
        case 12: go(k_tri_reg<D, 12, NW, NB, false, LA, true>); break;
        default: go(k_tri_reg<D, 16, NW, NB, false, LA, true>); break;
      }
    };
    using I0 = std::integral_constant<int, 0>;
    using I1 = std::integral_constant<int, 1>;
    using I2 = std::integral_constant<int, 2>;
    using ILA = std::integral_constant<int, REG_LA_DEV>;
    if constexpr (sizeof(D) != 8) {                                // complex: 15 warps, one buffer (or 7, two)
      if (nw == 15) {
        if (la > 0) by_w(std::integral_constant<int, 15>{}, I1{}, ILA{});
        else by_w(std::integral_constant<int, 15>{}, I1{}, I0{});
      } else {
        if (la > 0) by_w(std::integral_constant<int, 7>{}, I2{}, ILA{});
        else by_w(std::integral_constant<int, 7>{}, I2{}, I0{});
      }
    } else if (nw == 31) {
      if (la > 0) by_w(std::integral_constant<int, 31>{}, I1{}, ILA{});
      else by_w(std::integral_constant<int, 31>{}, I1{}, I0{});
    } else if (nw == 23) {
      if (la > 0) by_w(std::integral_constant<int, 23>{}, I1{}, ILA{});
      else by_w(std::integral_constant<int, 23>{}, I1{}, I0{});
    } else {
      if (la > 0) by_w(std::integral_constant<int, 15>{}, I2{}, ILA{});
      else by_w(std::integral_constant<int, 15>{}, I2{}, I0{});
    }
    CK(cudaGetLastError());
  }
}

template <typename D>
// xpm (one right-hand side, register kernel): DOWN writes the level's result to
// the U-packed buffer S.xU instead of x (coalesced stores; E_l z1 reads it there,
// Engine::apply_from); UP then takes x's old values from S.xU as they are.
static void launch_trisolve(Ctx *ctx, const StageDev<D> &S, int mode, const D *rhs, D *x, D *tmp,
                            const FArgs<D> &fa, const int *doneflag, int kc, int lvl = 0, int nr = 1, int64_t ldx = 0,
                            bool xpm = false, bool rhs_packed = false) {
  if (S.nblk <= 0 || S.rows == 0) return;
  if (nr > 1 && !(S.reg && S.mcap >= nr && (mode == TRI_DOWN || S.nf >= 0)))
    throw Error{GEMSLR_ERR_STATE, "several right-hand sides need the register-prefetched trisolve"};
  const CsrDev<D> *F = fa.F;
  const int64_t Fbase = fa.Fbase;
  const int64_t *Fp = F ? F->ptr : nullptr;
  const int32_t *Fc = F ? F->col : nullptr;
  const D *Fv = F ? F->val : nullptr;
  const int pgrid = grid_for((S.rows + 255) / 256, 4);
  if (S.reg) {
    const size_t smem = reg_smem_bytes<D>(S.Rg.ring, S.Rg.max_slices, S.Rg.imp_L + S.Rg.imp_U,
                                          S.Rg.plev_L + S.Rg.plev_U, S.reg_q > 1);
    RegDev<D> Rg = S.Rg;
    Rg.ldx = Rg.rsL = Rg.rsU = 0;
    D *rL = const_cast<D *>(S.Rg.rhsL), *rUp = S.rhs_up;
    if (nr > 1) {                                                 // per-column packed buffers
      rL = S.mL;
      rUp = S.mUp;
      Rg.mid = S.mU;
      Rg.ldx = ldx;
      Rg.rsL = Rg.rsU = std::max(S.lslices, S.uslices) * 32;
    }
    Rg.rhsL = rL;
    if (xpm && mode == TRI_DOWN && nr == 1) Rg.xP = S.xU;
    {
      // (profiler: a pack is timed and counted only when a kernel is launched)
      auto tp = [&]() { return Timed(ctx->prof, ctx->stream, KC_PACK); };
      if (mode == TRI_DOWN && rhs_packed && nr == 1) {
        // the packed right-hand side was written by the previous k_ewx (npk / pkpos)
      } else if (mode == TRI_DOWN) {
        const int64_t np = S.lslices * 32;
        const Timed tt = tp();
        launch_pdl(k_pack_gather<D>, dim3(grid_for((np + 255) / 256, 4), nr), dim3(256), 0, ctx->stream, np,
                   (const int *)S.lrow, rhs, rL, doneflag, (int64_t)ldx, (int64_t)Rg.rsL);
      } else if (S.nf >= 0) {
        Rg.rhsL = rUp;
        // one column: k_tri_reg updates x in place from its U-packed copy xU
        // (no tmp, no x -= tmp pass); several columns keep the tmp path
        const bool inpl = nr == 1 && S.xU != nullptr;
        const int64_t npu = inpl && !xpm ? S.uslices * 32 : 0;      // xpm: S.xU already holds z1 (DOWN)
        if (inpl) Rg.xU = S.xU;
        const int64_t work = std::max<int64_t>(S.nf, npu);
        if (work > 0) {
          const Timed tt = tp();
          launch_pdl(k_pack_f<D>, dim3(grid_for((work + 255) / 256, 4), nr), dim3(256), 0, ctx->stream, (int64_t)S.nf,
                     (const int *)S.fpos, (const int *)S.frow, Fp, Fc, Fv, (const D *)x, (int64_t)fa.nloc, fa.yh,
                     (int64_t)fa.nh, fa.yl, rUp, doneflag, (int64_t)ldx, (int64_t)Rg.rsL, npu, S.urow, S.xU);
        }
      } else {
        const Timed tt = tp();
        k_pack_rhs<D><<<pgrid, 256, 0, ctx->stream>>>(S.rows, S.row0, S.P.lpos, const_cast<D *>(S.Rg.rhsL), nullptr, Fp, Fc,
                                                      Fv, Fbase, x, fa.nloc, fa.yh, fa.nh, fa.yl, doneflag);
      }
    }
    Timed t(ctx->prof, ctx->stream, kc, lvl);
    Rg.dbg = (kc == KC_TRI_DOWN && lvl == g_tri_dbg_level) ? g_tri_dbg : nullptr;
    auto go = [&](auto kern, int nw) {
      static std::set<const void *> attr;                          // once per instance
      if (attr.insert((const void *)kern).second)
        CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 232448 - 1024));   // room for the static block info
      if (S.reg_q > 1) launch_pdl_cluster(kern, dim3(S.nblk * S.reg_q, nr), dim3(32 * (nw + 1)), smem, ctx->stream, S.reg_q,
                                          Rg, mode, x, tmp, doneflag);      // + the import warp
      else launch_pdl(kern, dim3(S.nblk, nr), dim3(32 * nw), smem, ctx->stream, Rg, mode, x, tmp, doneflag);
    };
    auto by_w = [&](auto nwc, auto nbc) {
      constexpr int NW = decltype(nwc)::value, NB = decltype(nbc)::value;
      auto by_la = [&](auto spc) {                                 // look-ahead (REG_LA new columns) or not
        constexpr bool SP = decltype(spc)::value;
        if (S.reg_la > 0) {
          switch (S.reg_w) {
            case 4: go(k_tri_reg<D, 4, NW, NB, SP, REG_LA_DEV>, NW); break;
            case 8: go(k_tri_reg<D, 8, NW, NB, SP, REG_LA_DEV>, NW); break;
            case 10: go(k_tri_reg<D, 10, NW, NB, SP, REG_LA_DEV>, NW); break;
            case 12: go(k_tri_reg<D, 12, NW, NB, SP, REG_LA_DEV>, NW); break;
            default: go(k_tri_reg<D, 16, NW, NB, SP, REG_LA_DEV>, NW); break;
          }
          return;
        }
        switch (S.reg_w) {
          case 4: go(k_tri_reg<D, 4, NW, NB, SP>, NW); break;
          case 8: go(k_tri_reg<D, 8, NW, NB, SP>, NW); break;
          case 10: go(k_tri_reg<D, 10, NW, NB, SP>, NW); break;
          case 12: go(k_tri_reg<D, 12, NW, NB, SP>, NW); break;
          default: go(k_tri_reg<D, 16, NW, NB, SP>, NW); break;
        }
      };
      if (S.reg_q > 1) by_la(std::true_type{});                    // split form: a cluster per block
      else by_la(std::false_type{});
    };
    using I1 = std::integral_constant<int, 1>;
    using I2 = std::integral_constant<int, 2>;
    // two record buffers where the register budget of NW warps holds them, one
    // for the wide variants (measured, C5/C4)
    if constexpr (sizeof(D) == 8) {
      if (S.reg_nw == 23) by_w(std::integral_constant<int, 23>{}, I1{});
      else by_w(std::integral_constant<int, 15>{}, I2{});
    } else {
      if (S.reg_nw == 15) by_w(std::integral_constant<int, 15>{}, I1{});
      else by_w(std::integral_constant<int, 7>{}, I2{});
    }
    CK(cudaGetLastError());
    return;
  }
  if (S.pipe) {
    const size_t smem = pipe_smem_bytes<D>(S.P.ring);
    static bool attr_set = false;
    if (!attr_set) {
      CK(cudaFuncSetAttribute(k_tri_pipe<D, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      CK(cudaFuncSetAttribute(k_tri_pipe<D, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      attr_set = true;
    }
    {
      Timed tp(ctx->prof, ctx->stream, KC_PACK);
      k_pack_rhs<D><<<pgrid, 256, 0, ctx->stream>>>(S.rows, S.row0, S.P.lpos, S.P.rhsL, mode == TRI_DOWN ? rhs : nullptr,
                                                    Fp, Fc, Fv, Fbase, x, fa.nloc, fa.yh, fa.nh, fa.yl, doneflag);
    }
    Timed t(ctx->prof, ctx->stream, kc, lvl);
    long long *dbg = kc == KC_TRI_DOWN ? g_tri_dbg : nullptr;
    if (S.far > 0)
      k_tri_pipe<D, true><<<S.nblk, 32 * (PIPE_NW_DEV + 1), smem, ctx->stream>>>(S.P, S.blk, mode, rhs, x, tmp, Fp, Fc, Fv, Fbase, doneflag, dbg);
    else
      k_tri_pipe<D, false><<<S.nblk, 32 * (PIPE_NW_DEV + 1), smem, ctx->stream>>>(S.P, S.blk, mode, rhs, x, tmp, Fp, Fc, Fv, Fbase, doneflag, dbg);
    CK(cudaGetLastError());
    return;
  }
  // level-per-barrier kernel (blobs that do not fit a pipeline stage; cluster option)
  if (mode == TRI_UP) {                                       // t = F_l y_J into tmp first
    Timed tp(ctx->prof, ctx->stream, KC_PACK);
    k_pack_rhs<D><<<pgrid, 256, 0, ctx->stream>>>(S.rows, S.row0, nullptr, tmp, nullptr, Fp, Fc, Fv, Fbase, x, fa.nloc,
                                                  fa.yh, fa.nh, fa.yl, doneflag);
    Fp = nullptr;
  }
  Timed t(ctx->prof, ctx->stream, kc, lvl);
  if (S.cps <= 1) {
    k_trisolve<D, false><<<S.nblk, 256, 0, ctx->stream>>>(S.L, S.U, S.blk, mode, rhs, x, tmp, Fp, Fc, Fv, Fbase, doneflag);
  } else {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(S.nblk * S.cps);
    cfg.blockDim = dim3(256);
    cfg.dynamicSmemBytes = 0;
    cfg.stream = ctx->stream;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = S.cps;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    CK(cudaLaunchKernelEx(&cfg, k_trisolve<D, true>, S.L, S.U, S.blk, mode, rhs, x, tmp, Fp, Fc, Fv, Fbase, doneflag));
  }
  CK(cudaGetLastError());
}

template <typename T>
void Engine<T>::spmv(const D *x, D *y, int mode, const D *b, const int *doneflag) {
  if (dist && n_bd >= 0 && sell_wmax <= 8 && !ctx->comm.hostmode()) {
    // Overlapped form (NCCL): pack the send values, fork the grouped send/recv onto
    // comm_stream, the interior slices meanwhile, join, then the slices with halo
    // columns.  Captured into the FGMRES graphs like the rest (fork / join events).
    if (!comm_stream) {
      CK(cudaStreamCreateWithFlags(&comm_stream, cudaStreamNonBlocking));
      CK(cudaEventCreateWithFlags(&ev_fork, cudaEventDisableTiming));
      CK(cudaEventCreateWithFlags(&ev_join, cudaEventDisableTiming));
    }
    const bool peers = !hA.peer.empty();
    if (peers) exchange(hA, x, doneflag, comm_stream);             // exterior columns (Note N P:L59-61)
    if (peers) CK(cudaEventRecord(ev_join, comm_stream));
    Timed t(ctx->prof, ctx->stream, KC_SPMV);
    constexpr int SPW = sizeof(D) == 8 ? 2 : 1;                  // (as below)
    auto part = [&](auto kern, const int *lst, int64_t cnt) {
      if (cnt <= 0) return;
      const int g2 = (int)std::max<int64_t>((cnt + 8 * SPW - 1) / (8 * SPW), 1);
      launch_pdl(kern, dim3(g2), dim3(256), 0, ctx->stream, n, cnt, sell_off, sell_col, sell_val, x, hA.rbuf, y, mode, b,
                 doneflag, lst);
    };
    part(k_spmv_sell2<D, false, SPW, 8>, sl_in, n_in);
    if (peers) CK(cudaStreamWaitEvent(ctx->stream, ev_join, 0));
    part(k_spmv_sell2<D, true, SPW, 8>, sl_bd, n_bd);
    CK(cudaGetLastError());
    return;
  }
  exchange(hA, x, doneflag);                                     // exterior columns (Note N P:L59-61)
  Timed t(ctx->prof, ctx->stream, KC_SPMV);
  if (use_wpr) {                                                  // long / uneven rows: a warp per row
    const int grid = grid_for((n + 7) / 8, 8);
    if (hA.nrecv > 0)
      launch_pdl(k_spmv_wpr<D, true>, dim3(grid), dim3(256), 0, ctx->stream, n, csr_ptr, csr_col, csr_val, x, hA.rbuf, y,
                 mode, b, doneflag);
    else
      launch_pdl(k_spmv_wpr<D, false>, dim3(grid), dim3(256), 0, ctx->stream, n, csr_ptr, csr_col, csr_val, x, hA.rbuf, y,
                 mode, b, doneflag);
    CK(cudaGetLastError());
    return;
  }
  if (sell_wmax <= 8) {                                           // 7-point / 5-point stencils and similar
    // two slices per warp for fp64; one for complex (two held 150 registers, one CTA per SM:
    // C4 SpMV 86.8 -> 66.8 us, 4.1 -> 5.4 TB/s, with one)
    constexpr int SPW = sizeof(D) == 8 ? 2 : 1;
    const int g2 = (int)std::max<int64_t>((nslices + 8 * SPW - 1) / (8 * SPW), 1);
    if (hA.nrecv > 0)
      launch_pdl(k_spmv_sell2<D, true, SPW, 8>, dim3(g2), dim3(256), 0, ctx->stream, n, nslices, sell_off, sell_col,
                 sell_val, x, hA.rbuf, y, mode, b, doneflag, (const int *)nullptr);
    else
      launch_pdl(k_spmv_sell2<D, false, SPW, 8>, dim3(g2), dim3(256), 0, ctx->stream, n, nslices, sell_off, sell_col,
                 sell_val, x, hA.rbuf, y, mode, b, doneflag, (const int *)nullptr);
    CK(cudaGetLastError());
    return;
  }
  const int grid = (int)((nslices + 7) / 8);
  if (hA.nrecv > 0)
    k_spmv_sell<D, true><<<std::max(grid, 1), 256, 0, ctx->stream>>>(n, nslices, sell_off, sell_col, sell_val, x, hA.rbuf,
                                                                    y, mode, b, doneflag);
  else
    k_spmv_sell<D, false><<<std::max(grid, 1), 256, 0, ctx->stream>>>(n, nslices, sell_off, sell_col, sell_val, x, hA.rbuf,
                                                                     y, mode, b, doneflag);
  CK(cudaGetLastError());
}

// DCGS2 pre-packing: the update pass of step j also writes u_{j+1} at its level-0 DOWN
// positions, so step j + 1's apply skips k_pack_gather (tail form at level 0, single pass)
template <typename T>
bool Engine<T>::prepack_ok() const {
  static const bool off = getenv("GEMSLR_NO_PREPACK") != nullptr;
  return !off && !lev.empty() && root_its == 0 && lev[0].st.tail && lev[0].st.tpos != nullptr && lev[0].o0 == 0;
}

// Alg. 2, single pass, from level l0: input `in` and output `out`
// are local vectors of which the local positions [lo_{l0}, n) are used.
template <typename T>
void Engine<T>::apply_from(int l0, const D *in, D *out, const int *doneflag, bool in_packed) {
  const int L = (int)lev.size();
  cudaStream_t s = ctx->stream;
  if (l0 == 0 && root_its > 0 && L > 0 && !dist) {                // Alg. 2 with GMRES at the root (NEXT-1)
    LevelDev<D> &d = lev[0];
    launch_trisolve(ctx, d.st, TRI_DOWN, in, out, tmp, FArgs<D>{}, doneflag, KC_TRI_DOWN, 0);   // z1
    {
      Timed t(ctx->prof, s, KC_EW);                              // z2 = b2 - E_0 z1 -> r[J_0]
      launch_ew<D>(s, d.s, d.o1, d.E.ptr, d.E.col, d.E.val, out, hE[0].rbuf, (int64_t)kHaloE, in, r, d.W, d.ldw, 0, partial,
                   tickets + 0, tvec, doneflag);
    }
    root_gmres(r + d.o1, out + d.o1, doneflag);                   // y2 ≈ Ŝ_0^-1 z2
    FArgs<D> fa;                                                   // y1 = z1 - U^-1 L^-1 F_0 y2
    fa.F = &d.F;
    fa.Fbase = d.o0;
    fa.nloc = n;
    fa.yh = hF[0].rbuf;
    fa.nh = hF[0].nrecv;
    launch_trisolve(ctx, d.st, TRI_UP, (const D *)nullptr, out, tmp, fa, doneflag, KC_TRI_UP, 0);
    return;
  }
  bool packed = in_packed && l0 == 0 && prepack_ok();             // this level's rhs already packed (k_ewx / k_dgs_upd)
  for (int l = l0; l < L; ++l) {
    LevelDev<D> &d = lev[l];
    const D *src = (l == l0) ? in : r;
    // z1 = U_l^-1 L_l^-1 b1  -> out[I_l] (xpm: U-packed in d.st.xU, read by E_l and the UP)
    const bool xpm = d.Ecol_p != nullptr;
    if (d.st.tail) launch_tail(ctx, d.st, true, src, out, FArgs<D>{}, doneflag, KC_TRI_DOWN, l, packed);
    else launch_trisolve(ctx, d.st, TRI_DOWN, src, out, tmp, FArgs<D>{}, doneflag, KC_TRI_DOWN, l, 1, 0, xpm, packed);
    packed = false;
    D *zp = d.st.tail ? d.st.tz : d.st.xU;                         // z1 in U-packed order (xpm)
    const D *zsrc = xpm ? (const D *)zp : (const D *)out;
    const int32_t *ecol = xpm ? d.Ecol_p : d.E.col;
    const int64_t znloc = kHaloE;                                  // E's halo columns start there (U-packed ones may exceed n)
    if (d.s > 0 || dist) {
      if (xpm) exchange(hE[l], zp, doneflag, nullptr, d.esidx_p);   // z1 entries of E_l's exterior columns
      else exchange(hE[l], out, doneflag);
      if (!dist && d.k > 0) {                                      // one cooperative launch: K6 + K7 + K8
        Timed t(ctx->prof, s, KC_EW);
        StageDev<D> &nst = (l + 1 < L) ? lev[l + 1].st : last;
        launch_ewx<D>(s, d.s, d.o1, d.E.ptr, ecol, d.E.val, zsrc, hE[l].rbuf, znloc, src, r, d.W, d.ldw, d.k, d.G,
                      partial, tickets + 0, tvec, ewflag, doneflag, d.npk, d.pkpos, nst.rhs_packed_buf(),
                      gtickets + l);
        packed = d.npk > 0;
        continue;
      }
      // z2 = b2 - E_l z1 ; this rank's part of s = W^H z2
      {
        Timed t(ctx->prof, s, KC_EW);
        launch_ew<D>(s, d.s, d.o1, d.E.ptr, ecol, d.E.val, zsrc, hE[l].rbuf, znloc, src, r, d.W, d.ldw, d.k, partial,
                     tickets + 0, tvec, doneflag);
      }
      if (d.k > 0) {                                              // u2 + z2, G s formed in every CTA
        if (dist) {
          if (d.s == 0) CK(cudaMemsetAsync(tvec, 0, d.k * sizeof(D), s));
          allreduce(tvec, d.k);                                   // W^H all-reduce
        }
        Timed t(ctx->prof, s, KC_WAXPY);
        const int grid = grid_for((std::max<int64_t>(d.s, 1) + 255) / 256, 8);
        StageDev<D> &nst = (l + 1 < L) ? lev[l + 1].st : last;
        k_waxpy<D><<<grid, 256, 0, s>>>(d.s, d.o1, d.W, d.ldw, d.k, d.G, tvec, r, doneflag, d.npk, d.pkpos,
                                        nst.rhs_packed_buf());
        packed = d.npk > 0;
        CK(cudaGetLastError());
      }
    }
  }
  // bottom: C_{L-1}^{-1} by block-Jacobi ILU, replicated on every rank
  const D *src = (l0 == L) ? in : r;
  const int64_t lL = plan.lo[L], nown = n - lL;
  if (!dist) {
    launch_trisolve(ctx, last, TRI_DOWN, src + lL, out + lL, tmp, FArgs<D>{}, doneflag, KC_TRI_LAST, 0, 1, 0, false,
                    packed);
  } else {
    CK(cudaMemsetAsync(rl_full, 0, plan.slast * sizeof(D), s));
    if (nown > 0)
      k_scatter_idx<D><<<grid_for((nown + 255) / 256, 2), 256, 0, s>>>(nown, last_idx_d, src + lL, rl_full, doneflag);
    allreduce(rl_full, plan.slast);                               // gather r_last (zeros elsewhere)
    launch_trisolve(ctx, last, TRI_DOWN, rl_full, yl_full, tmp, FArgs<D>{}, doneflag, KC_TRI_LAST);
    if (nown > 0)
      k_gather_idx<D><<<grid_for((nown + 255) / 256, 2), 256, 0, s>>>(nown, last_idx_d, yl_full, out + lL, doneflag);
  }
  // up: y1 = z1 - U^-1 L^-1 F_l y2
  for (int l = L - 1; l >= l0; --l) {
    LevelDev<D> &d = lev[l];
    exchange(hF[l], out, doneflag);                               // y entries of F_l's exterior columns
    FArgs<D> fa;
    fa.F = &d.F;
    fa.Fbase = d.o0;
    fa.nloc = n;
    fa.yh = hF[l].rbuf;
    fa.nh = hF[l].nrecv;
    fa.yl = yl_full;
    if (d.st.tail) launch_tail(ctx, d.st, false, (const D *)nullptr, out, fa, doneflag, KC_TRI_UP, l, false);
    else launch_trisolve(ctx, d.st, TRI_UP, (const D *)nullptr, out, tmp, fa, doneflag, KC_TRI_UP, l, 1, 0,
                         d.Ecol_p != nullptr);
  }
}

// ----------------------------------------------------------------- several right-hand sides (NEXT-4)
// apply / SpMV on n x nr blocks: the triangular
// solves of all columns run in ONE launch per stage (grid nblk x nr, every CTA
// streams the same factor records, so columns 2..nr read them from L2), the
// SpMV reads A once for all columns; the E/W coupling runs per column.
template <typename T>
bool Engine<T>::multi_ok() const {
  if (dist) return false;
  for (const auto &d : lev)
    if (!(d.st.nblk == 0 || d.st.rows == 0 || (d.st.reg && d.st.nf >= 0))) return false;
  return last.nblk == 0 || last.rows == 0 || last.reg;
}

template <typename T>
void Engine<T>::ensure_multi(int nr, int64_t ld) {
  Pool &P = ctx->pool;
  cudaStream_t s = ctx->stream;
  auto grow = [&](StageDev<D> &S) {
    if (!S.reg || S.mcap >= nr) return;
    const int64_t rs = std::max(S.lslices, S.uslices) * 32;
    S.mL = P.get<D>(std::max<int64_t>(rs * nr, 1));
    S.mU = P.get<D>(std::max<int64_t>(rs * nr, 1));
    S.mUp = P.get<D>(std::max<int64_t>(rs * nr, 1));
    CK(cudaMemsetAsync(S.mUp, 0, std::max<int64_t>(rs * nr, 1) * sizeof(D), s));   // UP rhs: zero off the F rows
    S.mcap = nr;
  };
  for (auto &d : lev) grow(d.st);
  grow(last);
  if (multi_cap < (int64_t)nr * ld) {
    rM = P.get<D>((size_t)nr * ld);
    tmpM = P.get<D>((size_t)nr * ld);
    multi_cap = (int64_t)nr * ld;
  }
}

template <typename T>
void Engine<T>::ew_column(LevelDev<D> &d, int l, const D *src, const D *z, D *dst, const int *doneflag) {
  cudaStream_t s = ctx->stream;
  Timed t(ctx->prof, s, KC_EW);
  if (d.k > 0) {
    launch_ewx<D>(s, d.s, d.o1, d.E.ptr, d.E.col, d.E.val, z, hE[l].rbuf, (int64_t)kHaloE, src, dst, d.W, d.ldw, d.k, d.G, partial,
                  tickets + 0, tvec, ewflag, doneflag, 0, nullptr, nullptr);   // no next-stage packing here
    return;
  }
  launch_ew<D>(s, d.s, d.o1, d.E.ptr, d.E.col, d.E.val, z, hE[l].rbuf, (int64_t)kHaloE, src, dst, d.W, d.ldw, 0, partial, tickets + 0,
               tvec, doneflag);
}

template <typename T>
void Engine<T>::apply_multi(const D *in, D *out, int64_t ld, int nr) {
  ensure_multi(nr, ld);
  const int L = (int)lev.size();
  for (int l = 0; l < L; ++l) {
    LevelDev<D> &d = lev[l];
    const D *src = (l == 0) ? in : rM;
    launch_trisolve(ctx, d.st, TRI_DOWN, src, out, tmpM, FArgs<D>{}, nullptr, KC_TRI_DOWN, l, nr, ld);
    if (d.s > 0)
      for (int c = 0; c < nr; ++c) ew_column(d, l, src + (size_t)c * ld, out + (size_t)c * ld, rM + (size_t)c * ld);
  }
  const D *src = (L == 0) ? in : rM;
  const int64_t lL = plan.lo[L];
  launch_trisolve(ctx, last, TRI_DOWN, src + lL, out + lL, tmpM, FArgs<D>{}, nullptr, KC_TRI_LAST, 0, nr, ld);
  for (int l = L - 1; l >= 0; --l) {
    LevelDev<D> &d = lev[l];
    FArgs<D> fa;
    fa.F = &d.F;
    fa.Fbase = d.o0;
    fa.nloc = n;
    launch_trisolve(ctx, d.st, TRI_UP, (const D *)nullptr, out, tmpM, fa, nullptr, KC_TRI_UP, l, nr, ld);
  }
}

template <typename T>
void Engine<T>::spmv_multi(const D *x, D *y, int64_t ld, int nr) {
  Timed t(ctx->prof, ctx->stream, KC_SPMV);
  const int grid = (int)std::max<int64_t>((nslices + 7) / 8, 1);
  if (sell_wmax <= 8)
    k_spmv_multi<D, 8><<<grid, 256, 0, ctx->stream>>>(n, nslices, sell_off, sell_col, sell_val, x, y, ld, nr);
  else if (sell_wmax <= 16)
    k_spmv_multi<D, 16><<<grid, 256, 0, ctx->stream>>>(n, nslices, sell_off, sell_col, sell_val, x, y, ld, nr);
  else
    for (int c = 0; c < nr; ++c) spmv(x + (size_t)c * ld, y + (size_t)c * ld, 0, nullptr, nullptr);
  CK(cudaGetLastError());
}

// ----------------------------------------------------------------- NEXT-1 root GMRES
// y2 ≈ Ŝ_0^-1 z2 by root_its steps of GMRES (x0 = 0) right-preconditioned by
// P(v) = C_0^-1 (v + W_0 G_0 W_0^H v) in the flexible form x = Z y, CGS2 and
// Givens as the outer FGMRES, early stop only on breakdown (oracle.cpp
// root_gmres).  Ŝ_0 t = C_0 t - E_0 U^-1 L^-1 F_0 t is formed as
// rows J_0 of Â [-(LU)^-1 F_0 t ; t]: an UP trisolve of level 0 on the vector
// [0 ; t] and a full SpMV.  Device-resident state, no host synchronisation (so
// it is captured in the FGMRES graphs); the inner kernels check an inner done
// flag that starts as the outer one.
template <typename T>
void Engine<T>::root_gmres(const D *bJ, D *xJ, const int *doneflag) {
  cudaStream_t s = ctx->stream;
  Pool &P = ctx->pool;
  LevelDev<D> &d0 = lev[0];
  const int m = root_its;
  const int64_t o1 = d0.o1, s0 = n - o1;
  if (!Vr) {
    ldr = (n + 31) / 32 * 32;
    Vr = P.get<D>((size_t)ldr * (m + 1));
    Zr = P.get<D>((size_t)ldr * m);
    wr = P.get<D>(ldr);
    ur = P.get<D>(ldr);
    zerov = P.get<D>(ldr);
    Hr = P.get<D>((size_t)(m + 1) * m);
    gr = P.get<D>(m + 1);
    snr = P.get<D>(m);
    yr = P.get<D>(m);
    rres = P.get<D>(3 * (GS_MAXC + 2));
    csr = P.get<double>(m);
    dblr = P.get<double>(8);
    histr = P.get<double>(m + 2);
    intsr = P.get<int>(4);
    doner = P.get<int>(1);
    skipr = P.get<int>(1);
    CK(cudaMemsetAsync(Zr, 0, (size_t)ldr * m * sizeof(D), s));
    CK(cudaMemsetAsync(Vr, 0, (size_t)ldr * (m + 1) * sizeof(D), s));
    CK(cudaMemsetAsync(zerov, 0, (size_t)ldr * sizeof(D), s));
    CK(cudaMemsetAsync(ur, 0, (size_t)ldr * sizeof(D), s));
  }
  FgmDev<D> f{doner, intsr, dblr, histr, Hr, gr, csr, snr};
  D *r1 = rres, *r2 = rres + (GS_MAXC + 2), *r3 = rres + 2 * (GS_MAXC + 2);
  const int g1 = grid_for((s0 + 255) / 256, 4);
  gs_pass(nullptr, 0, s0, 0, const_cast<D *>(bJ), 0, 0, nullptr, r1, 10, doneflag);   // ||z2||^2
  CK(cudaMemsetAsync(Hr, 0, (size_t)(m + 1) * m * sizeof(D), s));
  k_root_start<D><<<1, 32, 0, s>>>(f, m, r1, doneflag, skipr);
  k_scale<D><<<g1, 256, 0, s>>>(s0, bJ, Vr + o1, dblr + 4, doner);                   // V_0 = z2 / beta
  for (int j = 0; j < m; ++j) {
    D *vj = Vr + (size_t)j * ldr, *zj = Zr + (size_t)j * ldr;
    ew_column(d0, 0, vj, zerov, ur, doner);                                            // u = v + W G W^H v (E·0)
    apply_from(1, ur, zj, doner);                                                       // Z_j = C_0^-1 u
    CK(cudaMemsetAsync(zj, 0, (size_t)o1 * sizeof(D), s));                             // [0 ; Z_j]
    FArgs<D> fa;
    fa.F = &d0.F;
    fa.Fbase = d0.o0;
    fa.nloc = n;
    launch_trisolve(ctx, d0.st, TRI_UP, (const D *)nullptr, zj, tmp, fa, doner, KC_TRI_UP, 0);   // [-(LU)^-1 F Z_j ; Z_j]
    spmv(zj, wr, 0, nullptr, doner);                                                    // w[J_0] = Ŝ_0 Z_j
    gs_pass(Vr + o1, ldr, s0, j + 1, wr + o1, 0, 1, nullptr, r1, 10, doner);
    gs_pass(Vr + o1, ldr, s0, j + 1, wr + o1, 1, 1, r1, r2, 11, doner);
    gs_pass(Vr + o1, ldr, s0, j + 1, wr + o1, 1, 0, r2, r3, 12, doner);
    k_fgmres_col<D><<<1, 32, 0, s>>>(f, m, j, r1, r2, r3);
    if (j + 1 < m) k_scale<D><<<g1, 256, 0, s>>>(s0, wr + o1, Vr + (size_t)(j + 1) * ldr + o1, dblr + 2, doner);
  }
  k_root_solve<D><<<1, 32, 0, s>>>(f, m, skipr, yr);
  CK(cudaMemsetAsync(xJ, 0, (size_t)s0 * sizeof(D), s));
  k_xupdate<D><<<g1, 256, 0, s>>>(s0, Zr + o1, ldr, m, yr, xJ);                      // y2 = Z y
  CK(cudaGetLastError());
}

// Ĝ_l v = E_l (L_l U_l)^{-1} F_l C_l^{-1} v.  bufA[J_l] holds v
// on entry; on exit bufB[J_l] = Ĝ_l v.  bufA is used as scratch.
template <typename T>
void Engine<T>::ghat(int l, D *bufA, D *bufB) {
  LevelDev<D> &d = lev[l];
  cudaStream_t s = ctx->stream;
  // c = C_l^{-1} v  -> bufB[J_l]
  apply_from(l + 1, bufA, bufB, nullptr);
  // bufB[I_l] = 0 - U^-1 L^-1 F_l c = -u
  CK(cudaMemsetAsync(bufB + d.o0, 0, (d.o1 - d.o0) * sizeof(D), s));
  exchange(hF[l], bufB, nullptr);
  FArgs<D> fa;
  fa.F = &d.F;
  fa.Fbase = d.o0;
  fa.nloc = n;
  fa.yh = hF[l].rbuf;
  fa.nh = hF[l].nrecv;
  fa.yl = yl_full;
  launch_trisolve(ctx, d.st, TRI_UP, (const D *)nullptr, bufB, tmp, fa, nullptr, KC_TRI_UP);
  // bufB[J_l] = 0 - E_l (-u) = E_l u   (K6+K7 with k = 0, src = 0)
  exchange(hE[l], bufB, nullptr);
  launch_ew<D>(s, d.s, d.o1, d.E.ptr, d.E.col, d.E.val, bufB, hE[l].rbuf, (int64_t)kHaloE, (const D *)nullptr, bufB,
               (const D *)nullptr, 0, 0, partial, tickets + 1, tvec, nullptr);
}

template <typename T>
void Engine<T>::gs_pass(const D *Vb, int64_t ldvv, int64_t nn, int ncols, D *wv, int upd, int dot, const D *h_in,
                        D *resv, int ticket, const int *doneflag) {
  Timed t(ctx->prof, ctx->stream, KC_GS);
  // 13 values of V in flight per thread whatever the number of columns
  auto go = [&](auto kern, int tr) {
    const int grid = grid_for((nn + 32 * tr - 1) / (32 * tr), 3);
    launch_pdl(kern, dim3(grid), dim3(256), 0, ctx->stream, nn, Vb, ldvv, ncols, wv, upd, dot, h_in, partial,
               tickets + ticket, resv, doneflag);
  };
  static const bool old_gs = getenv("GEMSLR_OLD_GS") != nullptr;
  auto go2 = [&](auto kern) {
    const int grid = grid_for((nn + 255) / 256, ncols * (int)sizeof(D) <= 256 ? 2 : 1);
    launch_pdl(kern, dim3(grid), dim3(256), 0, ctx->stream, nn, Vb, ldvv, ncols, wv, upd, dot, h_in, partial,
               tickets + ticket, resv, doneflag);
  };
  bool done2 = false;
  if (!old_gs) {
    // measured on C5 (ncu, per pass): the warp-tile kernel sized to the column
    // count up to 32 columns (≈ 90 % of HBM), the column-split k_gs from 33 to
    // 48, the half-warp k_gs2h above (k_gs <1,13> is 2x slower there)
    done2 = true;
    constexpr int TU8 = sizeof(D) == 8 ? 4 : 1, TU16 = sizeof(D) == 8 ? 2 : 1;   // tiles in flight per warp (complex: registers)
    if (ncols <= 8) go2(k_gs2<D, 8, TU8, true>);
    else if (ncols <= 16) go2(k_gs2<D, 16, TU16, true>);
    else if (ncols <= 24) go2(k_gs2<D, 24>);
    else if (ncols <= 32) go2(k_gs2<D, 32>);
    else if constexpr (sizeof(D) == 8) {
      if (ncols > 48 && ncols <= 64) {
        const int grid = grid_for((nn + 127) / 128, 2);
        launch_pdl(k_gs2h<D>, dim3(grid), dim3(256), 0, ctx->stream, nn, Vb, ldvv, ncols, wv, upd, dot, h_in, partial,
                   tickets + ticket, resv, doneflag);
      } else {
        done2 = false;
      }
    } else {
      // complex: lane groups (2 x 32 or 4 x 26 columns per row tile)
      auto go3 = [&](auto kern, int rw, int per_sm = 1) {
        const int grid = grid_for((nn + 8 * rw - 1) / (8 * rw), per_sm);
        launch_pdl(kern, dim3(grid), dim3(256), 0, ctx->stream, nn, Vb, ldvv, ncols, wv, upd, dot, h_in, partial,
                   tickets + ticket, resv, doneflag);
      };
      if (ncols <= 48) done2 = false;                             // k_gs<2,6> measured faster here
      else if (ncols <= 64) go3(k_gs2g<D, 2, 32>, 16);
      else if (ncols <= 104) {
        static const int g8 = getenv("GEMSLR_GS2G") ? atoi(getenv("GEMSLR_GS2G")) : 4;
        if (g8 == 8) go3(k_gs2g<D, 8, 13>, 4, 2);                   // 8 groups of 4 lanes, 2 CTAs per SM
        else go3(k_gs2g<D, 4, 26>, 8);
      }
      else done2 = false;
    }
  }
  if (done2) {
  } else if (ncols <= 8) go(k_gs<D, 8, 1>, 8);
  else if (ncols <= 24) go(k_gs<D, 4, 3>, 4);
  else if (ncols <= 48) {
    // 33-48 columns, per pass (ncu on C5, 40-column cycle): dots only k_gs<4,6> (88 us at
    // 33 columns), update + dots k_gs<2,6> (127), update + norm the warp-tile k_gs2<48> (105;
    // k_gs's update needs a cross-warp sum per row tile through shared memory)
    if constexpr (sizeof(D) == 8) {
      if (!upd) {
        const int grid = grid_for((nn + 127) / 128, 2);            // 97 registers: 2 CTAs per SM
        launch_pdl(k_gs<D, 4, 6>, dim3(grid), dim3(256), 0, ctx->stream, nn, Vb, ldvv, ncols, wv, upd, dot, h_in,
                   partial, tickets + ticket, resv, doneflag);
      } else if (dot) {
        go(k_gs<D, 2, 6>, 2);                                      // (the warp-tile k_gs2<48> measured 1.5 % slower here)
      } else {
        const int grid = grid_for((nn + 255) / 256, 1);
        launch_pdl(k_gs2<D, 48, 1, false>, dim3(grid), dim3(256), 0, ctx->stream, nn, Vb, ldvv, ncols, wv, upd, dot,
                   h_in, partial, tickets + ticket, resv, doneflag);
      }
    } else {
      go(k_gs<D, 2, 6>, 2);
    }
  }
  else go(k_gs<D, 1, 13>, 1);
  CK(cudaGetLastError());
  allreduce(resv, dot ? ncols + 1 : 1);                          // dots and norms over ranks
  CK(cudaGetLastError());
}

// Step j of FGMRES with DCGS2 (c5', reading Q38): the dot pass over V_{0:j}, u_j = V_j
// and w (its last CTA completes column j - 1), then the update pass forming v_j and
// u_{j+1} = V_{j+1} (its last CTA takes the stopping decision).  fin: the closing dot
// pass of a cycle (w = u_jend, column jend - 1 completed, no update).  Several ranks:
// the dots and the norm are all-reduced between the passes and the two
// scalar steps run as one-warp kernels after them.
template <typename T>
void Engine<T>::dgs_step(int j, int m, int fin, const int *doneflag) {
  cudaStream_t st = ctx->stream;
  FgmDev<D> f{done, ints, dbl, hist, H, g, cs, sn};
  DcgDev<D> dd{f, Hraw, dcs};
  const int fuse = dist ? 0 : 1;
  D *u = V + (size_t)j * ldv;
  {
    Timed t(ctx->prof, st, KC_GS);
    const D *wv = fin ? u : w;
    // few columns: warp tiles holding every column of their rows (k_dgs_dotw); more:
    // column groups of up to 32 (k_dgs_dot), the columns dealt to the groups in turn
    auto gow = [&](auto kern, int tu, int per_sm, int nc) {
      const int ncg = std::max(1, (j + nc - 1) / nc);
      const int grid = grid_for((n + 256 * tu - 1) / (256 * tu), per_sm);
      if ((size_t)(2 * j + 3) * grid > partial_cap) throw Error{GEMSLR_ERR_INVALID_ARG, "DCGS2 partial buffer"};
      launch_pdl(kern, dim3(grid, ncg), dim3(256), 0, st, n, (const D *)V, ldv, j, (const D *)u, wv, partial,
                 tickets + 13, res, doneflag, dd, m, fin, fuse);
    };
    // (measured on C5 / C4 cycles, ncu: warp tiles in column groups of 8 or 16 for every j
    // re-read u and w per group and took 5.66 / 47.5 ms per cycle against 4.48 / 37.0 for
    // this split; warp tiles up to 32 columns 5.08 / 38.6)
    const int jw = sizeof(D) == 8 ? 16 : 8;                       // warp tiles up to jw columns
    auto goc = [&](auto kern, int npw, int tr) {
      const int ncg = std::max(1, (j + 8 * npw - 1) / (8 * npw));
      const int64_t nsteps = (n + 32 * tr - 1) / (32 * tr);
      // every CTA of every group resident at once (2 per SM): a rounded-up count left one CTA
      // for a second wave and doubled the pass at 3 column groups (C4, 65-96 columns)
      // (3 CTAs per SM at 80 registers measured slower: 1.73 against 1.58 ms per C5 cycle)
      const int nrb = (int)std::max<int64_t>(1, std::min<int64_t>(nsteps, (2 * num_sm()) / ncg));
      if ((size_t)(2 * j + 3) * nrb > partial_cap) throw Error{GEMSLR_ERR_INVALID_ARG, "DCGS2 partial buffer"};
      launch_pdl(kern, dim3(nrb, ncg), dim3(256), 0, st, n, (const D *)V, ldv, j, (const D *)u, wv, partial,
                 tickets + 13, res, doneflag, dd, m, fin, fuse);
    };
    if constexpr (sizeof(D) == 8) {
      if (j <= 8) gow(k_dgs_dotw<D, 8, 4>, 4, 2, 8);
      else if (j <= jw) gow(k_dgs_dotw<D, 16, 2>, 2, 1, 16);
    } else {
      if (j <= jw) gow(k_dgs_dotw<D, 8, 2>, 2, 1, 8);
    }
    if (j > jw) {
      if constexpr (sizeof(D) == 8) {
        // 33-48 columns in one group of 6 per warp (C5 cycle: 2.08 -> 1.86 ms of dot passes there)
        // (C5 cycle, dot passes: 8 rows per step with 4 or 2 columns per warp at 17-32 columns
        // 1.36 / 1.33 ms against 1.29; 2 x 8 at 9-16 columns 0.40 against 0.42 for dotw<16>)
        if (j > 32 && j <= 48) goc(k_dgs_dot<D, 6, 4>, 6, 4);
        else goc(k_dgs_dot<D, 4, 4>, 4, 4);
      } else {
        goc(k_dgs_dot<D, 4, 2>, 4, 2);   // (TR = 4 or 8 columns per warp measured slower on C4)
      }
    }
    CK(cudaGetLastError());
  }
  if (!fuse) {
    allreduce(res, 2 * j + 3);
    Timed t(ctx->prof, st, KC_FGM);
    launch_pdl(k_dgs_col<D>, dim3(1), dim3(32), 0, st, dd, m, j, fin, (const D *)res, doneflag);
    CK(cudaGetLastError());
  }
  if (fin) return;
  {
    Timed t(ctx->prof, st, KC_GS);
    const bool pk = prepack_ok() && j + 1 < m;
    // RPT = 2 rows per thread, all CTAs resident; C5 cycle: RPT 1 / 4 with 8-column batches
    // measured 5.05 / 4.73 ms against 4.69
    auto gou = [&](auto kern, int r, int per_sm) {
      const int grid = grid_for((n + 256 * r - 1) / (256 * r), per_sm);
      launch_pdl(kern, dim3(grid), dim3(256), 0, st, n, V, ldv, j, (const D *)w, (const D *)res, partial,
                 tickets + 14, doneflag, dd, m, fuse, pk ? lev[0].st.tpos : (const int *)nullptr,
                 pk ? lev[0].st.ntpos : (int64_t)0, pk ? lev[0].st.trhsL : (D *)nullptr);
    };
    // fp64: 2 rows x 16 columns per load batch, 2 CTAs per SM (124 registers); C5 cycle 4.50 ms
    // against 4.68 with 8-column batches (3 CTAs per SM), 4.75 / 5.43 with one row x 16
    if constexpr (sizeof(D) == 8) {
      gou(k_dgs_upd<D, 2, 16>, 2, 2);
    } else {
      gou(k_dgs_upd<D, 2, 8>, 2, 2);
    }
    CK(cudaGetLastError());
  }
  if (!fuse) {
    allreduce(dcs + 3, 1);
    Timed t(ctx->prof, st, KC_FGM);
    launch_pdl(k_dgs_check<D>, dim3(1), dim3(32), 0, st, dd, m, j, (const D *)res, doneflag);
    CK(cudaGetLastError());
  }
}

template <typename T>
double Engine<T>::norm(const D *x, int64_t nn, int ticket) {
  gs_pass(nullptr, 0, nn, 0, const_cast<D *>(x), 0, 0, nullptr, res, ticket, nullptr);
  D h;
  CK(cudaMemcpyAsync(&h, res, sizeof(D), cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  double v;
  if constexpr (std::is_same<D, double>::value) v = h; else v = h.x;
  return std::sqrt(std::max(v, 0.0));
}

// ----------------------------------------------------------------- small dense helpers (host)
template <typename S>
static bool inverse_small(int k, std::vector<S> &A) {    // Gauss-Jordan with partial pivoting, column-major
  std::vector<S> I((size_t)k * k, S(0));
  for (int i = 0; i < k; ++i) I[(size_t)i * k + i] = S(1);
  auto at = [&](std::vector<S> &M, int i, int j) -> S & { return M[(size_t)j * k + i]; };
  for (int c = 0; c < k; ++c) {
    int piv = c;
    for (int i = c + 1; i < k; ++i)
      if (absval(at(A, i, c)) > absval(at(A, piv, c))) piv = i;
    if (absval(at(A, piv, c)) == 0.0) return false;
    if (piv != c)
      for (int j = 0; j < k; ++j) { std::swap(at(A, c, j), at(A, piv, j)); std::swap(at(I, c, j), at(I, piv, j)); }
    const S d = at(A, c, c);
    for (int j = 0; j < k; ++j) { at(A, c, j) /= d; at(I, c, j) /= d; }
    for (int i = 0; i < k; ++i) {
      if (i == c) continue;
      const S f = at(A, i, c);
      if (f == S(0)) continue;
      for (int j = 0; j < k; ++j) { at(A, i, j) -= f * at(A, c, j); at(I, i, j) -= f * at(I, c, j); }
    }
  }
  A.swap(I);
  return true;
}

// ----------------------------------------------------------------- low rank (Arnoldi)
// Thick-restart (Krylov-Schur) Arnoldi on Ĝ_l, cycle length m = 2k,
// CGS2 orthogonalisation, Schur form of the projected matrix reordered so the
// k Ritz values with the largest |γ/(1-γ)| lead (
// reading Q6), converged when they change by < tol relatively between cycles
// (reading Q8).  Real A keeps a real basis: the selected set is
// closed under conjugation (a split pair takes k+1, reading Q7) and its
// invariant subspace gets a real orthonormal basis.  W = V Y, R = Y^H H Y,
// G = (I - R)^{-1} - I.  Built bottom-up l = L-1 .. 0.
template <typename T>
void Engine<T>::build_lowrank(const gemslr_params &prm, unsigned long long seed) {
  const int L = (int)lev.size();
  cudaStream_t s = ctx->stream;
  const bool is_real = std::is_same<T, double>::value;
  const double tol = prm.arnoldi_tol > 0 ? prm.arnoldi_tol : 1e-2;
  const int maxcyc = prm.arnoldi_max_cycles > 0 ? prm.arnoldi_max_cycles : 10;
  D *bufA = ctx->pool.get<D>(n + 1);
  D *bufB = ctx->pool.get<D>(n + 1);
  CK(cudaMemsetAsync(bufA, 0, (n + 1) * sizeof(D), s));
  CK(cudaMemsetAsync(bufB, 0, (n + 1) * sizeof(D), s));
  D *hres = ctx->pool.get<D>(3 * (GS_MAXC + 2));
  for (int l = L - 1; l >= 0; --l) {
    LevelDev<D> &d = lev[l];
    const int64_t sl = d.s;                                       // rows of J_l on this rank
    const int64_t sg = nglob - plan.st.o[l + 1];                  // rows of J_l on all ranks
    int k = prm.rank;
    if (k <= 0 || sg == 0) { d.k = 0; continue; }
    if (k > sg) k = (int)sg;
    int m = std::min<int64_t>(2 * (int64_t)k, sg);
    if (m < k + 1 && m < sg) m = k + 1;
    if (m + 1 > GS_MAXC) throw Error{GEMSLR_ERR_INVALID_ARG, "rank too large for the Arnoldi workspace (2k+1 > 104)"};
    const int64_t ld = (std::max<int64_t>(sl, 1) + 31) / 32 * 32;
    D *Vb = ctx->pool.get<D>((size_t)ld * (m + 1));
    D *Wt = ctx->pool.get<D>((size_t)ld * (k + 2));
    D *Yd = ctx->pool.get<D>((size_t)m * (k + 2));
    // start vector: uniform[-1,1] from the seed over the GLOBAL rows of J_l
    // (reading Q8), this rank's rows taken from it, normalised
    std::mt19937_64 rng(seed + 7919ull * (unsigned long long)(l + 1));
    std::uniform_real_distribution<double> U(-1.0, 1.0);
    std::vector<T> vg(sg);
    for (auto &e : vg) {
      if constexpr (std::is_same<T, double>::value) e = U(rng); else e = zc(U(rng), U(rng));
    }
    std::vector<T> v0(sl);
    for (int64_t i = 0; i < sl; ++i) v0[i] = vg[plan.gpos[d.o1 + i] - plan.st.o[l + 1]];
    if (sl > 0) CK(cudaMemcpyAsync(Vb, v0.data(), sl * sizeof(D), cudaMemcpyHostToDevice, s));
    double nv = norm(Vb, sl, 2);
    if (nv == 0.0) throw Error{GEMSLR_ERR_LOWRANK, "Arnoldi start vector is zero"};
    {
      std::vector<double> inv{1.0 / nv};
      double *dsc = ctx->pool.get<double>(1);
      CK(cudaMemcpyAsync(dsc, inv.data(), sizeof(double), cudaMemcpyHostToDevice, s));
      k_scale<D><<<grid_for((sl + 255) / 256, 4), 256, 0, s>>>(sl, Vb, Vb, dsc, nullptr);
    }
    // H: (m+1) x m host, column-major
    std::vector<zc> H((size_t)(m + 1) * m, zc(0));
    auto Hat = [&](int i, int j) -> zc & { return H[(size_t)j * (m + 1) + i]; };
    int j0 = 0, cyc = 0, kk = 0;
    std::vector<zc> prev_sel;
    std::vector<zc> Yh, Rk;
    bool converged = false;
    double *dscale = ctx->pool.get<double>(1);
    while (true) {
      ++cyc;
      int mm = m;
      bool breakdown = false;
      double hlast = 0;
      for (int j = j0; j < m; ++j) {
        D *vj = Vb + (size_t)j * ld;
        CK(cudaMemcpyAsync(bufA + d.o1, vj, sl * sizeof(D), cudaMemcpyDeviceToDevice, s));
        ghat(l, bufA, bufB);
        D *wv = bufB + d.o1;
        gs_pass(Vb, ld, sl, j + 1, wv, 0, 1, nullptr, hres, 3, nullptr);
        gs_pass(Vb, ld, sl, j + 1, wv, 1, 1, hres, hres + (GS_MAXC + 2), 4, nullptr);
        gs_pass(Vb, ld, sl, j + 1, wv, 1, 0, hres + (GS_MAXC + 2), hres + 2 * (GS_MAXC + 2), 5, nullptr);
        std::vector<T> hh(3 * (GS_MAXC + 2));
        CK(cudaMemcpyAsync(hh.data(), hres, hh.size() * sizeof(D), cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        const double eta = std::sqrt(std::max(0.0, std::real(zc(hh[j + 1]))));
        const double hn = std::sqrt(std::max(0.0, std::real(zc(hh[2 * (GS_MAXC + 2)]))));
        for (int i = 0; i <= j; ++i) Hat(i, j) = zc(hh[i]) + zc(hh[(GS_MAXC + 2) + i]);
        Hat(j + 1, j) = hn;
        hlast = hn;
        if (!(hn > 1e-14 * eta) || !std::isfinite(hn)) { mm = j + 1; breakdown = true; break; }
        const double inv = 1.0 / hn;
        CK(cudaMemcpyAsync(dscale, &inv, sizeof(double), cudaMemcpyHostToDevice, s));
        k_scale<D><<<grid_for((sl + 255) / 256, 4), 256, 0, s>>>(sl, wv, Vb + (size_t)(j + 1) * ld, dscale, nullptr);
        CK(cudaStreamSynchronize(s));
      }
      // Schur of the mm x mm projected matrix
      std::vector<zc> Hm((size_t)mm * mm), Tm((size_t)mm * mm), Q((size_t)mm * mm);
      for (int j = 0; j < mm; ++j)
        for (int i = 0; i < mm; ++i) Hm[(size_t)j * mm + i] = Hat(i, j);
      if (!schur_complex(mm, Hm.data(), Tm.data(), Q.data()))
        throw Error{GEMSLR_ERR_LOWRANK, "Schur iteration did not converge at level " + std::to_string(l)};
      // select the k largest |γ/(1-γ)|
      std::vector<int> idx(mm);
      std::vector<double> key(mm);
      for (int i = 0; i < mm; ++i) {
        const zc gm = Tm[(size_t)i * mm + i];
        key[i] = std::abs(gm / (zc(1.0) - gm));
        idx[i] = i;
      }
      std::stable_sort(idx.begin(), idx.end(), [&](int a, int b) { return key[a] > key[b]; });
      int want = std::min(k, mm);
      std::vector<char> sel(mm, 0);
      for (int i = 0; i < want; ++i) sel[idx[i]] = 1;
      if (is_real) {                                    // never split a conjugate pair (Q7)
        for (int i = 0; i < mm; ++i) {
          if (!sel[i]) continue;
          const zc gi = Tm[(size_t)i * mm + i];
          if (std::abs(gi.imag()) <= 1e-12 * std::max(1.0, std::abs(gi))) continue;
          int best = -1;
          double bd = 1e300;
          for (int q = 0; q < mm; ++q) {
            if (q == i) continue;
            double dd = std::abs(Tm[(size_t)q * mm + q] - std::conj(gi));
            if (dd < bd) { bd = dd; best = q; }
          }
          if (best >= 0 && !sel[best] && bd <= 1e-6 * std::max(1.0, std::abs(gi))) sel[best] = 1;
        }
      }
      for (int i = 0; i < mm; ++i)
        if (sel[i] && std::abs(zc(1.0) - Tm[(size_t)i * mm + i]) < 1e-12)
          throw Error{GEMSLR_ERR_LOWRANK, "Ritz value within 1e-12 of 1 at level " + std::to_string(l)};
      schur_reorder(mm, Tm.data(), Q.data(), sel);
      int ks = 0;
      for (char c : sel) ks += c;
      // convergence of the selected Ritz values (sorted by key)
      std::vector<zc> cur(ks);
      for (int i = 0; i < ks; ++i) cur[i] = Tm[(size_t)i * mm + i];
      std::sort(cur.begin(), cur.end(), [](const zc &a, const zc &b) {
        double ka = std::abs(a / (zc(1.0) - a)), kb = std::abs(b / (zc(1.0) - b));
        if (ka != kb) return ka > kb;
        if (a.real() != b.real()) return a.real() < b.real();
        return a.imag() < b.imag();
      });
      if (!prev_sel.empty() && prev_sel.size() == cur.size()) {
        double worst = 0;
        for (int i = 0; i < ks; ++i) worst = std::max(worst, std::abs(cur[i] - prev_sel[i]) / std::max(std::abs(cur[i]), 1e-300));
        converged = worst < tol;
      }
      if (breakdown || mm <= ks) converged = true;
      prev_sel = cur;
      // basis Y (mm x kk) of the selected invariant subspace
      std::vector<zc> Yc((size_t)mm * ks);
      for (int c = 0; c < ks; ++c)
        for (int i = 0; i < mm; ++i) Yc[(size_t)c * mm + i] = Q[(size_t)c * mm + i];
      if (is_real) {                                    // real orthonormal basis of span(Y)
        std::vector<std::vector<double>> cand;
        for (int c = 0; c < ks; ++c) {
          std::vector<double> re(mm), im(mm);
          for (int i = 0; i < mm; ++i) { re[i] = Yc[(size_t)c * mm + i].real(); im[i] = Yc[(size_t)c * mm + i].imag(); }
          cand.push_back(re);
          cand.push_back(im);
        }
        std::vector<std::vector<double>> basis;
        for (auto &v : cand) {
          double n0 = 0;
          for (double e : v) n0 += e * e;
          n0 = std::sqrt(n0);
          if (n0 == 0) continue;
          for (int pass = 0; pass < 2; ++pass)
            for (auto &b : basis) {
              double dd = 0;
              for (int i = 0; i < mm; ++i) dd += b[i] * v[i];
              for (int i = 0; i < mm; ++i) v[i] -= dd * b[i];
            }
          double n1 = 0;
          for (double e : v) n1 += e * e;
          n1 = std::sqrt(n1);
          if (n1 <= 1e-8 * n0) continue;
          for (double &e : v) e /= n1;
          basis.push_back(v);
          if ((int)basis.size() == ks) break;
        }
        if ((int)basis.size() != ks) throw Error{GEMSLR_ERR_LOWRANK, "real invariant-subspace basis is rank deficient"};
        for (int c = 0; c < ks; ++c)
          for (int i = 0; i < mm; ++i) Yc[(size_t)c * mm + i] = zc(basis[c][i], 0.0);
      }
      kk = ks;
      // Rk = Y^H H_mm Y
      Rk.assign((size_t)kk * kk, zc(0));
      {
        std::vector<zc> HY((size_t)mm * kk, zc(0));
        for (int c = 0; c < kk; ++c)
          for (int j = 0; j < mm; ++j) {
            const zc y = Yc[(size_t)c * mm + j];
            if (y == zc(0)) continue;
            for (int i = 0; i < mm; ++i) HY[(size_t)c * mm + i] += Hm[(size_t)j * mm + i] * y;
          }
        for (int c = 0; c < kk; ++c)
          for (int a = 0; a < kk; ++a) {
            zc acc = 0;
            for (int i = 0; i < mm; ++i) acc += std::conj(Yc[(size_t)a * mm + i]) * HY[(size_t)c * mm + i];
            Rk[(size_t)c * kk + a] = acc;
          }
      }
      Yh = Yc;
      // W (or the restarted basis) = V_mm Y  -> Wt
      {
        std::vector<T> Yt((size_t)mm * kk);
        for (size_t i = 0; i < Yt.size(); ++i) {
          if constexpr (std::is_same<T, double>::value) Yt[i] = Yc[i].real(); else Yt[i] = Yc[i];
        }
        CK(cudaMemcpyAsync(Yd, Yt.data(), Yt.size() * sizeof(D), cudaMemcpyHostToDevice, s));
        k_gemm_tall<D><<<grid_for((sl + 255) / 256, 4), 256, 0, s>>>(sl, Vb, ld, mm, Yd, kk, Wt, ld);
        CK(cudaGetLastError());
      }
      if (converged || cyc >= maxcyc) break;
      // thick restart: V[:, 0:kk] = V Y ; V[:, kk] = v_{m+1} ; H = [Rk ; hlast * Y[mm-1, :]]
      CK(cudaMemcpyAsync(Vb, Wt, (size_t)ld * kk * sizeof(D), cudaMemcpyDeviceToDevice, s));
      CK(cudaMemcpyAsync(Vb + (size_t)kk * ld, Vb + (size_t)mm * ld, sl * sizeof(D), cudaMemcpyDeviceToDevice, s));
      std::fill(H.begin(), H.end(), zc(0));
      for (int c = 0; c < kk; ++c) {
        for (int a = 0; a < kk; ++a) Hat(a, c) = Rk[(size_t)c * kk + a];
        Hat(kk, c) = hlast * Yc[(size_t)c * mm + (mm - 1)];
      }
      j0 = kk;
      CK(cudaStreamSynchronize(s));
    }
    CK(cudaStreamSynchronize(s));
    d.cycles = cyc;
    d.k = kk;
    d.ldw = ld;
    d.W = Wt;
    // G = (I - Rk)^{-1} - I
    using S = typename std::conditional<std::is_same<T, double>::value, double, zc>::type;
    std::vector<S> IR((size_t)kk * kk), Rs((size_t)kk * kk);
    for (int c = 0; c < kk; ++c)
      for (int a = 0; a < kk; ++a) {
        zc v = Rk[(size_t)c * kk + a];
        S sv;
        if constexpr (std::is_same<S, double>::value) sv = v.real(); else sv = v;
        Rs[(size_t)c * kk + a] = sv;
        IR[(size_t)c * kk + a] = (a == c ? S(1) : S(0)) - sv;
      }
    if (!inverse_small(kk, IR)) throw Error{GEMSLR_ERR_LOWRANK, "I - R singular at level " + std::to_string(l)};
    for (int a = 0; a < kk; ++a) IR[(size_t)a * kk + a] -= S(1);
    d.Gh = IR;
    d.Rh = Rs;
    d.G = ctx->pool.upload<D>(IR, s);
    // host copy of W for export
    d.Wh.assign((size_t)sl * kk, S(0));
    for (int c = 0; c < kk; ++c)
      CK(cudaMemcpyAsync(d.Wh.data() + (size_t)c * sl, Wt + (size_t)c * ld, sl * sizeof(D), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
  }
}

// ----------------------------------------------------------------- FGMRES
template <typename T>
void Engine<T>::ensure_krylov(int m, int maxit) {
  if (kry_m >= m && hist_cap >= maxit + 1) return;
  Pool &P = ctx->pool;
  ldv = (n + 31) / 32 * 32;
  if (kry_m < m) {
    V = P.get<D>((size_t)ldv * (m + 1));
    Z = P.get<D>((size_t)ldv * m);
    w = P.get<D>(n + 1);
    H = P.get<D>((size_t)(m + 1) * m);
    g = P.get<D>(m + 1);
    sn = P.get<D>(m);
    cs = P.get<double>(m);
    ydev = P.get<D>(m + 1);
    dbl = P.get<double>(8);
    ints = P.get<int>(8);
    done = P.get<int>(2);
    Hraw = P.get<D>((size_t)(m + 1) * m);
    dcs = P.get<D>(4);
    kry_m = m;
  }
  if (hist_cap < maxit + 1) {
    // the captured iteration graphs hold this pointer (graph_hist): allocate with
    // room to spare so a later solve with a larger maxit rarely forces a re-capture
    const int cap = std::max(maxit + 1, std::max(4095, 2 * hist_cap));
    hist = P.get<double>(cap + 1);
    hist_cap = cap;
  }
}

// Right-preconditioned FGMRES(m) with CGS2 (c5 of DESIGN.md).
template <typename T>
int Engine<T>::solve(const D *b, D *x, double rtol, int m, int maxit, int *its_out, double *hist_out, int hcap,
                     int *hlen, double *frel) {
  cudaStream_t s = ctx->stream;
  if (m + 1 > GS_MAXC) throw Error{GEMSLR_ERR_INVALID_ARG, "restart must be <= 103"};
  struct Range {                                              // NVTX range for ncu --nvtx filtering
    Range() { nvtxRangePushA("gemslr_solve"); }
    ~Range() { nvtxRangePop(); }
  } nvtx_range;
  ensure_krylov(m, maxit);
  std::vector<double> hh;
  // ||b||, r = b - A x and ||r|| with one round trip (slot 4 of res is free here)
  double bnorm, beta;
  {
    D *rn = res + 3 * (GS_MAXC + 2);
    gs_pass(nullptr, 0, n, 0, const_cast<D *>(b), 0, 0, nullptr, rn, 6, nullptr);
    spmv(x, w, 1, b, nullptr);
    gs_pass(nullptr, 0, n, 0, w, 0, 0, nullptr, rn + 1, 6, nullptr);
    D h2[2];
    CK(cudaMemcpyAsync(h2, rn, 2 * sizeof(D), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    double v0, v1;
    if constexpr (std::is_same<D, double>::value) { v0 = h2[0]; v1 = h2[1]; } else { v0 = h2[0].x; v1 = h2[1].x; }
    bnorm = std::sqrt(std::max(v0, 0.0));
    beta = std::sqrt(std::max(v1, 0.0));
  }
  int its = 0;
  if (bnorm == 0.0) {
    k_fill<D><<<grid_for((n + 255) / 256, 4), 256, 0, s>>>(n, x, dzero<D>());
    if (hist_out && hcap > 0) hist_out[0] = 0.0;
    if (hlen) *hlen = 1;
    if (its_out) *its_out = 0;
    if (frel) *frel = 0.0;
    CK(cudaStreamSynchronize(s));
    return GEMSLR_OK;
  }
  hh.push_back(beta / bnorm);
  double *dsc = dbl + 4;
  FgmDev<D> f{done, ints, dbl, hist, H, g, cs, sn};
  const bool dcgs = ctx->orth == 1;
  while (beta > rtol * bnorm && its < maxit) {
    // V0 = r / beta ; g = (beta, 0, ...) ; state
    {
      double hv[8] = {bnorm, rtol, 0, 0, dcgs ? 1.0 : 1.0 / beta, 0, 0, 0};   // DCGS2: u_0 = r
      int iv[4] = {0, its, maxit, 0};
      CK(cudaMemcpyAsync(dbl, hv, sizeof(hv), cudaMemcpyHostToDevice, s));
      CK(cudaMemcpyAsync(ints, iv, sizeof(iv), cudaMemcpyHostToDevice, s));
      CK(cudaMemsetAsync(done, 0, 2 * sizeof(int), s));
      std::vector<D> g0(m + 1, dzero<D>());
      if (!dcgs) {                                                // DCGS2: g_0 = alpha from the first dot pass
        if constexpr (std::is_same<D, double>::value) g0[0] = beta; else g0[0] = D{beta, 0.0};
      }
      CK(cudaMemcpyAsync(g, g0.data(), (m + 1) * sizeof(D), cudaMemcpyHostToDevice, s));
      CK(cudaMemsetAsync(H, 0, (size_t)(m + 1) * m * sizeof(D), s));
      if (dcgs) CK(cudaMemsetAsync(Hraw, 0, (size_t)(m + 1) * m * sizeof(D), s));
      Timed t(ctx->prof, s, KC_UTIL);
      k_scale<D><<<grid_for((n + 255) / 256, 4), 256, 0, s>>>(n, w, V, dsc, nullptr);
    }
    D *res1 = res, *res2 = res + (GS_MAXC + 2), *res3 = res + 2 * (GS_MAXC + 2);
    std::vector<cudaEvent_t> evs;
    if (hflags_cap < m) {
      if (hflags) cudaFreeHost(hflags);
      hflags = nullptr;
      if (cudaMallocHost(&hflags, (size_t)m * sizeof(int)) != cudaSuccess) throw Error{GEMSLR_ERR_OOM, "pinned flags"};
      hflags_cap = m;
    }
    int j = 0;
    // one FGMRES iteration: every launch is on ctx->stream with fixed buffers,
    // so iteration j can be captured once as a CUDA graph and replayed
    auto iteration = [&](int jj) {
      cudaStream_t st = ctx->stream;
      D *vj = V + (size_t)jj * ldv;
      D *zj = Z + (size_t)jj * ldv;
      apply_from(0, vj, zj, done, dcgs && jj > 0);                // Z_j = M^{-1} V_j (DCGS2 j > 0: V_j pre-packed)
      spmv(zj, w, 0, nullptr, done);                              // w = A Z_j
      if (dcgs) {                                                 // (DCGS2: V_j holds u_j)
        dgs_step(jj, m, 0, done);
        return;
      }
      gs_pass(V, ldv, n, jj + 1, w, 0, 1, nullptr, res1, 7, done);  // h = V^H w, ||w||^2
      gs_pass(V, ldv, n, jj + 1, w, 1, 1, res1, res2, 8, done);     // w -= V h ; h2 = V^H w
      gs_pass(V, ldv, n, jj + 1, w, 1, 0, res2, res3, 9, done);     // w -= V h2 ; ||w||^2
      {
        Timed t(ctx->prof, st, KC_FGM);                          // Givens column + v_{j+1} = w / h_{j+1}
        launch_pdl(k_fgmres_scale<D>, dim3(grid_for((n + 255) / 256, 4)), dim3(256), 0, st, f, m, jj, res1, res2, res3,
                   n, w, V + (size_t)(jj + 1) * ldv);
        CK(cudaGetLastError());
      }
    };
    static const bool no_graph = getenv("GEMSLR_NO_GRAPH") != nullptr;
    // graphs on one GPU and over NCCL (its calls are captured with the kernels); the
    // host-staged backend synchronises inside its collectives and cannot be captured
    const bool use_graph = !no_graph && !ctx->comm.hostmode() && !ctx->prof.on;
    if (use_graph && (graph_m != m || graph_V != V || graph_hist != hist || graph_orth != ctx->orth)) {
      for (auto &ge : graphs) if (ge) cudaGraphExecDestroy(ge);
      graphs.assign(m, nullptr);
      graph_m = m;
      graph_V = V;
      graph_hist = hist;
      graph_orth = ctx->orth;
    }
    auto capture = [&](int jj) {                                 // capture on a private stream, replay on ours
      if (!cap_stream) CK(cudaStreamCreateWithFlags(&cap_stream, cudaStreamNonBlocking));
      cudaStream_t user = ctx->stream;
      ctx->stream = cap_stream;
      cudaGraph_t g = nullptr;
      CK(cudaStreamBeginCapture(cap_stream, cudaStreamCaptureModeRelaxed));
      try {
        iteration(jj);
      } catch (...) {
        cudaStreamEndCapture(cap_stream, &g);
        if (g) cudaGraphDestroy(g);
        ctx->stream = user;
        throw;
      }
      CK(cudaStreamEndCapture(cap_stream, &g));
      ctx->stream = user;
      CK(cudaGraphInstantiate(&graphs[jj], g, 0));
      cudaGraphDestroy(g);
    };
    if (use_graph)                                                // all m iterations captured before the first runs
      for (int jj = 0; jj < m; ++jj)
        if (!graphs[jj]) capture(jj);
    // the iteration that reaches maxit is known here: nothing is queued after it (the
    // done flag still ends the cycle earlier on convergence or breakdown)
    const int jmax = std::min(m, maxit - its);
    for (j = 0; j < jmax; ++j) {
      if (use_graph) {
        if (!graphs[j]) {                                         // (not reached: captured above)
          if (!cap_stream) CK(cudaStreamCreateWithFlags(&cap_stream, cudaStreamNonBlocking));
          cudaStream_t user = ctx->stream;
          ctx->stream = cap_stream;
          cudaGraph_t g = nullptr;
          CK(cudaStreamBeginCapture(cap_stream, cudaStreamCaptureModeRelaxed));
          try {
            iteration(j);
          } catch (...) {
            cudaStreamEndCapture(cap_stream, &g);
            if (g) cudaGraphDestroy(g);
            ctx->stream = user;
            throw;
          }
          CK(cudaStreamEndCapture(cap_stream, &g));
          ctx->stream = user;
          CK(cudaGraphInstantiate(&graphs[j], g, 0));
          cudaGraphDestroy(g);
        }
        CK(cudaGraphLaunch(graphs[j], s));
      } else {
        iteration(j);
      }
      // the done flag of iteration j reaches pinned host memory asynchronously;
      // the host reads it kLag iterations later, so the GPU always has the next
      // iterations queued (a synchronous copy would drain the stream; with a lag
      // of 2 a host hiccup of ~2 ms starved the GPU in some bench runs).  After
      // convergence at most kLag queued iterations run, every kernel exiting at once.
      // (profiling: lag 0, so no iteration is queued after the last one and every
      // timed launch is a real one)
      const int kLag = ctx->prof.on ? 0 : 6;
      CK(cudaMemcpyAsync(hflags + j, done, sizeof(int), cudaMemcpyDeviceToHost, s));
      cudaEvent_t e;
      CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      CK(cudaEventRecord(e, s));
      evs.push_back(e);
      if (j >= kLag) {
        CK(cudaEventSynchronize(evs[j - kLag]));
        if (((volatile int *)hflags)[j - kLag]) break;
      }
    }
    if (hstage_cap < 64) {
      if (hstage) cudaFreeHost(hstage);
      hstage = nullptr;
      if (cudaMallocHost(&hstage, 4096) != cudaSuccess) throw Error{GEMSLR_ERR_OOM, "pinned staging"};
      hstage_cap = 4096;
    }
    if (dcgs) {                                                   // the closing dot pass completes column jend - 1
      int *jh = reinterpret_cast<int *>(hstage);
      CK(cudaMemcpyAsync(jh, ints, 4 * sizeof(int), cudaMemcpyDeviceToHost, s));
      CK(cudaStreamSynchronize(s));
      dgs_step(jh[0], m, 1, nullptr);
    } else {
      CK(cudaStreamSynchronize(s));
    }
    for (auto e : evs) cudaEventDestroy(e);
    if (ctx->prof.on) {
      CK(cudaStreamSynchronize(s));
      ctx->prof.flush();
    }
    // the cycle's state in one round trip: counters, history entries, H and g into a
    // pinned staging buffer on the solver stream
    const size_t offH = 64 + (((size_t)m + 1) * sizeof(double) + 63) / 64 * 64;
    const size_t need = offH + ((size_t)(m + 1) * m + m + 1) * sizeof(D);
    if (hstage_cap < need) {
      if (hstage) cudaFreeHost(hstage);
      hstage = nullptr;
      if (cudaMallocHost(&hstage, need) != cudaSuccess) throw Error{GEMSLR_ERR_OOM, "pinned staging"};
      hstage_cap = need;
    }
    int *iv_h = reinterpret_cast<int *>(hstage);
    double *hist_h = reinterpret_cast<double *>(hstage + 64);
    const T *Hh = reinterpret_cast<const T *>(hstage + offH);
    const T *gh = Hh + (size_t)(m + 1) * m;
    const int hcnt = std::max(0, std::min(m, hist_cap - its));    // hist[its + 1 .. its + m] (within the buffer)
    CK(cudaMemcpyAsync(iv_h, ints, 4 * sizeof(int), cudaMemcpyDeviceToHost, s));
    if (hcnt > 0) CK(cudaMemcpyAsync(hist_h, hist + its + 1, hcnt * sizeof(double), cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(hstage + offH, H, (size_t)(m + 1) * m * sizeof(D), cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(hstage + offH + (size_t)(m + 1) * m * sizeof(D), g, (m + 1) * sizeof(D), cudaMemcpyDeviceToHost,
                       s));
    CK(cudaStreamSynchronize(s));
    const int jend = iv_h[0];
    const int its_new = iv_h[1];
    if (its_new - its > hcnt) throw Error{GEMSLR_ERR_CUDA, "history beyond the staged entries"};
    for (int q = 0; q < its_new - its; ++q) hh.push_back(hist_h[q]);
    its = its_new;
    // y = H[0:jend,0:jend]^{-1} g  (upper triangular after the rotations; host)
    std::vector<T> y(jend);
    for (int i = jend - 1; i >= 0; --i) {
      T acc = gh[i];
      for (int c = i + 1; c < jend; ++c) acc -= Hh[(size_t)c * (m + 1) + i] * y[c];
      y[i] = acc / Hh[(size_t)i * (m + 1) + i];
    }
    if (jend > 0) {
      CK(cudaMemcpyAsync(ydev, y.data(), jend * sizeof(D), cudaMemcpyHostToDevice, s));
      Timed t(ctx->prof, s, KC_UTIL);
      k_xupdate<D><<<grid_for((n + 255) / 256, 4), 256, 0, s>>>(n, Z, ldv, jend, ydev, x);   // x += Z y
      CK(cudaGetLastError());
    }
    spmv(x, w, 1, b, nullptr);                                    // explicit r = b - A x
    beta = norm(w, n, 6);
    if (jend == 0) break;
  }
  if (its_out) *its_out = its;
  const int hl = (int)hh.size();
  if (hlen) *hlen = std::min(hl, hcap);
  if (hist_out)
    for (int i = 0; i < hl && i < hcap; ++i) hist_out[i] = hh[i];
  if (frel) *frel = beta / bnorm;
  return beta > rtol * bnorm ? GEMSLR_NOT_CONVERGED : GEMSLR_OK;
}

// ----------------------------------------------------------------- bundle export
static void write_bin(const std::string &path, const void *p, size_t bytes) {
  FILE *f = std::fopen(path.c_str(), "wb");
  if (!f) throw Error{GEMSLR_ERR_INVALID_ARG, "cannot write " + path};
  if (bytes) std::fwrite(p, 1, bytes, f);
  std::fclose(f);
}

// Collective on every rank (several ranks: the W_l rows of all ranks are summed
// into the global J_l order by one all-reduce per level; rank 0 writes the bundle).
// The structure and R_l, G_l are replicated; the ILU factors are written by a
// single-rank context only (each rank holds its own blocks; the oracle recomputes
// every factor from its own A anyway, c3).
template <typename T>
void Engine<T>::export_bundle(const std::string &dir) const {
  using S = typename std::conditional<std::is_same<T, double>::value, double, zc>::type;
  const bool dist = plan.nranks > 1;
  std::vector<std::vector<S>> Wg(lev.size());
  for (int l = 0; l < (int)lev.size(); ++l) {
    const auto &d = lev[l];
    if (d.k == 0) continue;
    if (!dist) { Wg[l] = d.Wh; continue; }
    const int64_t og = plan.st.o[l + 1], sg = nglob - og;
    std::vector<S> full((size_t)sg * d.k, S(0));
    for (int c = 0; c < d.k; ++c)
      for (int64_t i = 0; i < d.s; ++i) full[(size_t)c * sg + (plan.gpos[d.o1 + i] - og)] = d.Wh[(size_t)c * d.s + i];
    D *buf = static_cast<D *>(ctx->alloc.alloc(std::max<size_t>(full.size(), 1) * sizeof(D)));
    try {
      CK(cudaMemcpyAsync(buf, full.data(), full.size() * sizeof(D), cudaMemcpyHostToDevice, ctx->stream));
      const_cast<Engine<T> *>(this)->allreduce(buf, full.size());
      CK(cudaMemcpyAsync(full.data(), buf, full.size() * sizeof(D), cudaMemcpyDeviceToHost, ctx->stream));
      CK(cudaStreamSynchronize(ctx->stream));
    } catch (...) {
      ctx->alloc.release(buf);
      throw;
    }
    ctx->alloc.release(buf);
    Wg[l].swap(full);
  }
  if (plan.rank != 0) return;
  mkdir(dir.c_str(), 0755);
  std::string man = "{\n";
  const char *vt = std::is_same<T, double>::value ? "float64" : "complex128";
  auto add = [&](const std::string &name, const char *dt, const void *p, size_t count, size_t esz, std::vector<int64_t> shape) {
    write_bin(dir + "/" + name + ".bin", p, count * esz);
    man += "  \"" + name + "\": {\"dtype\": \"" + dt + "\", \"shape\": [";
    for (size_t i = 0; i < shape.size(); ++i) man += (i ? ", " : "") + std::to_string(shape[i]);
    man += "]},\n";
  };
  const Structure &st = plan.st;
  add("perm", "int64", st.perm.data(), st.perm.size(), 8, {(int64_t)st.perm.size()});
  add("level_off", "int64", st.o.data(), st.o.size(), 8, {(int64_t)st.o.size()});
  for (int l = 0; l < st.L; ++l)
    add("blocks_" + std::to_string(l), "int64", st.blk[l].data(), st.blk[l].size(), 8, {(int64_t)st.blk[l].size()});
  add("last_off", "int64", st.last.data(), st.last.size(), 8, {(int64_t)st.last.size()});
  auto facs = [&](const std::string &tag, const std::vector<Factor<T>> &F) {
    for (int which = 0; which < 2; ++which) {
      std::vector<int64_t> ptr, nnzoff{0};
      std::vector<int32_t> col;
      std::vector<T> val;
      for (auto &f : F) {
        const Csr<T> &M = which ? f.U : f.L;
        ptr.insert(ptr.end(), M.ptr.begin(), M.ptr.end());
        col.insert(col.end(), M.col.begin(), M.col.end());
        val.insert(val.end(), M.val.begin(), M.val.end());
        nnzoff.push_back((int64_t)col.size());
      }
      const std::string b = tag + (which ? "_U" : "_L");
      add(b + "_ptr", "int64", ptr.data(), ptr.size(), 8, {(int64_t)ptr.size()});
      add(b + "_col", "int32", col.data(), col.size(), 4, {(int64_t)col.size()});
      add(b + "_val", vt, val.data(), val.size(), sizeof(T), {(int64_t)val.size()});
      add(b + "_nnzoff", "int64", nnzoff.data(), nnzoff.size(), 8, {(int64_t)nnzoff.size()});
    }
  };
  if (!dist) {
    for (int l = 0; l < st.L; ++l) facs("fac" + std::to_string(l), plan.fac[l]);
    facs("faclast", plan.lastfac);
  }
  std::string ranks = "[";
  for (int l = 0; l < (int)lev.size(); ++l) {
    const auto &d = lev[l];
    ranks += (l ? ", " : "") + std::to_string(d.k);
    if (d.k > 0) {
      add("W_" + std::to_string(l), vt, Wg[l].data(), Wg[l].size(), sizeof(T), {(int64_t)d.k, nglob - st.o[l + 1]});
      add("R_" + std::to_string(l), vt, d.Rh.data(), d.Rh.size(), sizeof(T), {(int64_t)d.k, (int64_t)d.k});
      add("G_" + std::to_string(l), vt, d.Gh.data(), d.Gh.size(), sizeof(T), {(int64_t)d.k, (int64_t)d.k});
    }
  }
  ranks += "]";
  const gemslr_params &p = ctx->params;
  man += "  \"meta\": {\"n\": " + std::to_string(n) + ", \"levels\": " + std::to_string(st.L) + ", \"dtype\": \"" + vt +
         "\", \"ilu\": " + std::to_string(p.ilu) + ", \"ilut_drop\": " + std::to_string(p.ilut_drop) +
         ", \"ilut_fill\": " + std::to_string(p.ilut_fill) + ", \"ranks\": " + ranks +
         ", \"nranks\": " + std::to_string(plan.nranks) + "}\n}\n";
  write_bin(dir + "/manifest.json", man.data(), man.size());
}

template <typename T>
std::string Engine<T>::stats_json() const {
  const Structure &st = plan.st;
  std::string j = "{";
  j += "\"n\": " + std::to_string(plan.Ahat.n) + ", \"nnz\": " + std::to_string(plan.Ahat.nnz());
  j += ", \"nnz_local\": " + std::to_string(plan.Aloc.nnz());
  j += ", \"levels\": " + std::to_string(st.L);
  j += ", \"level_off\": [";
  for (size_t i = 0; i < st.o.size(); ++i) j += (i ? ", " : "") + std::to_string(st.o[i]);
  j += "], \"fill\": " + std::to_string((double)plan.fac_nnz / std::max<int64_t>(1, plan.Ahat.nnz()));
  j += ", \"fac_nnz\": " + std::to_string(plan.fac_nnz);
  j += ", \"sell_padded\": " + std::to_string(sell_padded);
  j += std::string(", \"spmv_kernel\": \"") + (use_wpr ? "wpr" : (sell_wmax <= 8 ? "sell2" : "sell")) + "\"";
  auto stage = [&](const StageDev<D> &S) {
    return "{\"blocks\": " + std::to_string(S.nblk) + ", \"rows\": " + std::to_string(S.rows) + ", \"cps\": " +
           std::to_string(S.cps) + ", \"depth_L\": " + std::to_string(S.depthL) + ", \"depth_U\": " +
           std::to_string(S.depthU) + ", \"nnz\": " + std::to_string(S.nnz) + ", \"padded\": " + std::to_string(S.padded) +
           ", \"pipe\": " + (S.pipe ? "true" : "false") + ", \"chunks\": " + std::to_string(S.nchunks) +
           ", \"far\": " + std::to_string(S.far) + ", \"near\": " + std::to_string(S.nearc) +
           ", \"kernel\": \"" + (S.reg ? "reg" : S.pipe ? "pipe" : "level") + "\", \"reg_w\": " + std::to_string(S.reg_w) +
           ", \"split\": " + std::to_string(S.reg ? S.reg_q : 1) + ", \"reg_nw\": " + std::to_string(S.reg_nw) +
           ", \"la\": " + std::to_string(S.reg ? S.reg_la : 0) +
           ", \"reg_bytes\": " + std::to_string(S.reg_bytes) +
           ", \"tail\": " + (S.tail ? std::string("{\"rows\": ") + std::to_string(S.tail_rows) + ", \"bytes\": " +
                                       std::to_string(S.tail_bytes) + ", \"depth_down\": [" +
                                       std::to_string(S.depth_tail[0]) + ", " + std::to_string(S.depth_tail[1]) + ", " +
                                       std::to_string(S.depth_tail[2]) + "], \"depth_up\": [" +
                                       std::to_string(S.depth_tail[3]) + ", " + std::to_string(S.depth_tail[4]) + ", " +
                                       std::to_string(S.depth_tail[5]) + "], \"w\": [" + std::to_string(S.td_w) + ", " +
                                       std::to_string(S.tu_w) + "], \"nw\": [" + std::to_string(S.td_nw) + ", " +
                                       std::to_string(S.tu_nw) + "], \"la\": [" + std::to_string(S.td_la) + ", " +
                                       std::to_string(S.tu_la) + "], \"nnz\": [" + std::to_string(S.tail_nnz[0]) + ", " +
                                       std::to_string(S.tail_nnz[1]) + ", " + std::to_string(S.tail_nnz[2]) + ", " +
                                       std::to_string(S.tail_nnz[3]) + ", " + std::to_string(S.tail_nnz[4]) + "]}"
                                 : std::string("null")) + "}";
  };
  j += ", \"stages\": [";
  for (size_t l = 0; l < lev.size(); ++l) {
    const auto &d = lev[l];
    j += (l ? ", " : "") + std::string("{\"stage\": ") + stage(d.st) + ", \"s\": " + std::to_string(d.s) + ", \"k\": " +
         std::to_string(d.k) + ", \"cycles\": " + std::to_string(d.cycles) + ", \"nnzE\": " + std::to_string(d.E.nnz) +
         ", \"nnzF\": " + std::to_string(d.F.nnz) + "}";
  }
  j += "], \"last\": " + stage(last);
  j += ", \"packs\": [";                                          // host packing of every level stage
  for (size_t l = 0; l < plan.stage.size(); ++l) {
    const auto &R = plan.stage[l].reg;
    j += (l ? ", " : "") + std::string("{\"ok\": ") + (R.ok ? "true" : "false") + ", \"Q\": " + std::to_string(R.Q) +
         ", \"ring\": " + std::to_string(R.ring) + ", \"W\": " + std::to_string(R.W) + ", \"imp_L\": " +
         std::to_string(R.imp_L) + ", \"imp_U\": " + std::to_string(R.imp_U) + ", \"plev_L\": " +
         std::to_string(R.plev_L) + ", \"plev_U\": " + std::to_string(R.plev_U) + ", \"exports\": " +
         std::to_string(R.exports) + ", \"records\": " + std::to_string(R.nrec) + ", \"max_levels\": " +
         std::to_string(R.max_levels) + "}";
  }
  j += "]";
  j += ", \"setup_host_s\": " + std::to_string(setup_host_s) + ", \"setup_device_s\": " + std::to_string(setup_dev_s) +
       ", \"arnoldi_s\": " + std::to_string(arnoldi_s);
  j += ", \"device_bytes\": " + std::to_string(ctx->pool.bytes);
  int64_t hsend = plan.hA.nsend(), hrecv = plan.hA.nrecv();
  for (size_t l = 0; l < plan.hE.size(); ++l) {
    hsend += plan.hE[l].nsend() + plan.hF[l].nsend();
    hrecv += plan.hE[l].nrecv() + plan.hF[l].nrecv();
  }
  j += ", \"nranks\": " + std::to_string(plan.nranks) + ", \"rank\": " + std::to_string(plan.rank) +
       ", \"n_local\": " + std::to_string(plan.nloc) + ", \"halo_send\": " + std::to_string(hsend) +
       ", \"halo_recv\": " + std::to_string(hrecv) + ", \"allreduces\": " + std::to_string(ctx->comm.allreduces) +
       ", \"exchanges\": " + std::to_string(ctx->comm.exchanges);
  j += ", \"kernels\": {";
  bool first = true;
  for (int k = 0; k < KC_COUNT; ++k) {
    if (!first) j += ", ";
    first = false;
    j += "\"" + std::string(kKernelName[k]) + "\": {\"ms\": " + std::to_string(ctx->prof.ms[k]) + ", \"count\": " +
         std::to_string(ctx->prof.count[k]) + ", \"by_level\": [" + std::to_string(ctx->prof.sub_ms[k][0]) + ", " +
         std::to_string(ctx->prof.sub_ms[k][1]) + ", " + std::to_string(ctx->prof.sub_ms[k][2]) + ", " +
         std::to_string(ctx->prof.sub_ms[k][3]) + "]}";
  }
  j += "}}";
  return j;
}

template struct Engine<double>;
template struct Engine<zc>;

}  // namespace gemslr

// =================================================================== C-ABI
using namespace gemslr;

struct gemslr_ctx : public Ctx {};

static gemslr_status fail(const gemslr_ctx *c, int code, const std::string &msg) {
  if (c) const_cast<gemslr_ctx *>(c)->err = msg;
  return (gemslr_status)code;
}

template <typename F>
static gemslr_status guarded(gemslr_ctx *c, F &&fn) {
  try {
    if (c && c->device >= 0) {
      cudaError_t e = cudaSetDevice(c->device);
      if (e != cudaSuccess) return fail(c, GEMSLR_ERR_CUDA, std::string("cudaSetDevice: ") + cudaGetErrorString(e));
    }
    return fn();
  } catch (const Error &e) {
    return fail(c, e.code, e.msg);
  } catch (const std::bad_alloc &) {
    return fail(c, GEMSLR_ERR_OOM, "host allocation failed");
  } catch (const std::exception &e) {
    return fail(c, GEMSLR_ERR_INVALID_ARG, e.what());
  }
}

extern "C" {

static gemslr_status create_common(gemslr_ctx **out, int cuda_device, void *cuda_stream, gemslr_ctx **made) {
  if (!out) return GEMSLR_ERR_INVALID_ARG;
  *out = nullptr;
  auto *c = new gemslr_ctx();
  c->device = cuda_device;
  c->host_only = cuda_device < 0;
  c->stream = static_cast<cudaStream_t>(cuda_stream);
  c->pool.A = &c->alloc;
  if (!c->host_only) {
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || cuda_device >= ndev || cudaSetDevice(cuda_device) != cudaSuccess) {
      delete c;
      return GEMSLR_ERR_CUDA;
    }
  }
  *made = c;
  return GEMSLR_OK;
}

gemslr_status gemslr_create(gemslr_ctx **out, int cuda_device, void *nccl_comm, void *cuda_stream) {
  gemslr_ctx *c = nullptr;
  gemslr_status st = create_common(out, cuda_device, cuda_stream, &c);
  if (st) return st;
  if (nccl_comm) {
    if (c->host_only) { delete c; return GEMSLR_ERR_INVALID_ARG; }
    try {
      c->comm.borrow(nccl_comm, nullptr);
    } catch (const Error &e) {
      delete c;
      return (gemslr_status)e.code;
    }
  }
  *out = c;
  return GEMSLR_OK;
}

gemslr_status gemslr_nccl_unique_id(const char *nccl_lib, void *id128) {
  if (!id128) return GEMSLR_ERR_INVALID_ARG;
  try {
    void *h = Comm::open_lib(nccl_lib);
    auto f = reinterpret_cast<int (*)(void *)>(dlsym(h, "ncclGetUniqueId"));
    if (!f || f(id128) != 0) return GEMSLR_ERR_NCCL;
  } catch (const Error &e) {
    return (gemslr_status)e.code;
  }
  return GEMSLR_OK;
}

gemslr_status gemslr_create_dist(gemslr_ctx **out, int cuda_device, void *cuda_stream, int nranks, int rank,
                                 const void *nccl_id, const char *nccl_lib) {
  if (nranks < 1 || rank < 0 || rank >= nranks) return GEMSLR_ERR_INVALID_ARG;
  gemslr_ctx *c = nullptr;
  gemslr_status st = create_common(out, cuda_device, cuda_stream, &c);
  if (st) return st;
  c->comm.nranks = nranks;
  c->comm.rank = rank;
  if (!c->host_only && (nranks > 1 || nccl_id)) {
    if (!nccl_id) { delete c; return GEMSLR_ERR_INVALID_ARG; }
    try {
      c->comm.init(nccl_lib, nranks, rank, nccl_id);
      c->comm.force = nranks == 1;                                 // one rank: the distributed path over NCCL
    } catch (const Error &e) {
      delete c;
      return (gemslr_status)e.code;
    }
  }
  *out = c;
  return GEMSLR_OK;
}

gemslr_status gemslr_create_hostcomm(gemslr_ctx **out, int cuda_device, void *cuda_stream, int nranks, int rank,
                                     gemslr_allreduce_fn allreduce, gemslr_sendrecv_fn sendrecv, void *user) {
  if (nranks < 1 || rank < 0 || rank >= nranks || !allreduce || !sendrecv) return GEMSLR_ERR_INVALID_ARG;
  gemslr_ctx *c = nullptr;
  gemslr_status st = create_common(out, cuda_device, cuda_stream, &c);
  if (st) return st;
  c->comm.nranks = nranks;
  c->comm.rank = rank;
  c->comm.h_allreduce = allreduce;
  c->comm.h_sendrecv = sendrecv;
  c->comm.h_user = user;
  *out = c;
  return GEMSLR_OK;
}

gemslr_status gemslr_set_allocator(gemslr_ctx *c, void *(*alloc_fn)(size_t, void *), void (*free_fn)(void *, void *),
                                   void *user) {
  if (!c) return GEMSLR_ERR_INVALID_ARG;
  if (c->ready) return fail(c, GEMSLR_ERR_STATE, "set_allocator must precede setup");
  if ((alloc_fn == nullptr) != (free_fn == nullptr)) return fail(c, GEMSLR_ERR_INVALID_ARG, "alloc and free come in pairs");
  c->alloc.alloc_fn = alloc_fn;
  c->alloc.free_fn = free_fn;
  c->alloc.user = user;
  return GEMSLR_OK;
}

gemslr_status gemslr_set_coordinates(gemslr_ctx *c, int dim, const double *coords) {
  if (!c || dim < 0 || (dim > 0 && !coords)) return fail(c, GEMSLR_ERR_INVALID_ARG, "bad coordinates");
  if (c->ready) return fail(c, GEMSLR_ERR_STATE, "set_coordinates must precede setup");
  c->coord_dim = dim;
  c->coords_src = coords;   // n x dim doubles, copied by setup once n is known
  return GEMSLR_OK;
}

}  // extern "C"

template <typename T>
static gemslr_status do_setup(gemslr_ctx *c, std::unique_ptr<Engine<T>> &E, int64_t n, const int64_t *rowptr,
                              const int32_t *colidx, const void *values, const gemslr_params *prm) {
  E.reset(new Engine<T>());
  E->ctx = c;
  SetupOptions opt;
  opt.levels = prm->levels;
  opt.p = prm->subdomains;
  opt.ilu = prm->ilu;
  opt.tau = prm->ilut_drop;
  opt.lfil = prm->ilut_fill > 0 ? prm->ilut_fill : 10;
  opt.last_blocks = prm->last_blocks;
  opt.shift = prm->ilu_shift;
  opt.nranks = c->comm.nranks;
  opt.rank = c->comm.rank;
  // split form of the level-0 triangular solves (plan.hpp): only with the register
  // kernel (tri_kernel 0, no cluster override); GEMSLR_SPLIT=1/2/4 forces it
  opt.split = (prm->tri_kernel != 0 || prm->cluster_ctas > 0) ? 1 : prm->tri_split;
  if (getenv("GEMSLR_SPLIT")) opt.split = atoi(getenv("GEMSLR_SPLIT"));
  // tail form (DESIGN 6b): boundary rows last in every B_l and the tail sweeps; fp64 with
  // the register kernel (GEMSLR_TAIL=0 keeps the plain order and sweeps; =2 the order only)
  opt.tail = (prm->tri_kernel == 0 && prm->cluster_ctas <= 0) ? 1 : 0;
  if (opt.split > 1) opt.tail = 0;                                  // a forced split form keeps the plain order
  if (getenv("GEMSLR_TAIL")) opt.tail = opt.tail && atoi(getenv("GEMSLR_TAIL")) != 0;
  if (getenv("GEMSLR_TAIL_DIST")) opt.tail_dist = atoi(getenv("GEMSLR_TAIL_DIST"));   // experiments
  if (!c->host_only) opt.sms = num_sm();
  if (c->coord_dim > 0 && c->coords_src) {
    c->coords.assign(c->coords_src, c->coords_src + (size_t)n * c->coord_dim);
    opt.coord_dim = c->coord_dim;
    opt.coords = c->coords.data();
  }
  Error err{0, ""};
  auto t0 = std::chrono::steady_clock::now();
  if (!build_host_plan<T>(n, rowptr, colidx, static_cast<const T *>(values), opt, E->plan, err)) {
    E.reset();
    return fail(c, err.code, err.msg);
  }
  auto t1 = std::chrono::steady_clock::now();
  E->setup_host_s = std::chrono::duration<double>(t1 - t0).count();
  E->n = n;
  E->dist = E->plan.nranks > 1 || c->comm.force;
  if (c->host_only) return GEMSLR_OK;
  E->upload(c->stream);
  CK(cudaStreamSynchronize(c->stream));
  auto t2 = std::chrono::steady_clock::now();
  E->setup_dev_s = std::chrono::duration<double>(t2 - t1).count();
  E->build_lowrank(*prm, prm->seed);
  E->root_its = prm->root_inner_its;                              // NEXT-1 (after the low rank: Arnoldi uses l0 >= 1)
  CK(cudaStreamSynchronize(c->stream));
  E->arnoldi_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t2).count();
  return GEMSLR_OK;
}

extern "C" {


gemslr_status gemslr_setup(gemslr_ctx *c, gemslr_dtype dtype, int64_t n, const int64_t *rowptr, const int32_t *colidx,
                           const void *values, const gemslr_params *prm) {
  if (!c) return GEMSLR_ERR_INVALID_ARG;
  if (c->ready) return fail(c, GEMSLR_ERR_STATE, "setup called twice on one context");
  if (!rowptr || !colidx || !values || !prm || n <= 0) return fail(c, GEMSLR_ERR_INVALID_ARG, "null pointer or n <= 0");
  if (prm->levels < 1 || prm->subdomains < 1 || prm->rank < 0 || (dtype != GEMSLR_F64 && dtype != GEMSLR_C128) ||
      (prm->ilu != GEMSLR_ILU0 && prm->ilu != GEMSLR_ILUT) || prm->ilut_drop < 0)
    return fail(c, GEMSLR_ERR_INVALID_ARG, "levels < 1, subdomains < 1, rank < 0 or bad dtype/ilu");
  if (2 * prm->rank + 2 > GS_MAXC) return fail(c, GEMSLR_ERR_INVALID_ARG, "rank > 51 not supported (Arnoldi cycle 2k + 1 <= 103 columns)");
  if (prm->root_inner_its < 0 || prm->root_inner_its + 2 > GS_MAXC ||
      (prm->root_inner_its > 0 && (c->comm.nranks > 1 || c->comm.force)))
    return fail(c, GEMSLR_ERR_INVALID_ARG, "root_inner_its < 0, too large, or with several ranks (one GPU only)");
  if (prm->tri_split < 0 || prm->tri_split == 3 || prm->tri_split > 4)
    return fail(c, GEMSLR_ERR_INVALID_ARG, "tri_split must be 0, 1, 2 or 4");
  if (prm->ilu_shift != 0.0 && (dtype != GEMSLR_C128 || !(prm->ilu_shift == prm->ilu_shift)))
    return fail(c, GEMSLR_ERR_INVALID_ARG, "ilu_shift needs complex arithmetic (GEMSLR_C128)");
  c->params = *prm;
  gemslr_status st = guarded(c, [&]() -> gemslr_status {
    if (dtype == GEMSLR_F64) return do_setup<double>(c, c->ed, n, rowptr, colidx, values, prm);
    return do_setup<zc>(c, c->ez, n, rowptr, colidx, values, prm);
  });
  if (st == GEMSLR_OK) {
    c->ready = true;
    c->dtype = dtype;
  } else {
    c->ed.reset();
    c->ez.reset();
    c->pool.clear();
  }
  return st;
}

gemslr_status gemslr_layout(const gemslr_ctx *c, int64_t *n_local, int64_t *grow) {
  if (!c || !n_local) return GEMSLR_ERR_INVALID_ARG;
  if (!c->ready) return fail(c, GEMSLR_ERR_STATE, "layout before setup");
  auto go = [&](const auto &pl) {
    *n_local = pl.nloc;
    if (grow)
      for (int64_t i = 0; i < pl.nloc; ++i) grow[i] = pl.st.perm[pl.gpos[i]];
  };
  if (c->dtype == GEMSLR_F64) go(c->ed->plan); else go(c->ez->plan);
  return GEMSLR_OK;
}

// Halo plan of this rank (tests): which = 0 SpMV, 1 E_l, 2 F_l.  counts[2*nranks]:
// values sent to / received from each rank; sglob / rglob (may be NULL):
// global permuted positions, concatenated by peer in rank order.
gemslr_status gemslr_halo_plan(const gemslr_ctx *c, int which, int level, int64_t *counts, int64_t *sglob,
                               int64_t *rglob) {
  if (!c || !counts || which < 0 || which > 2) return GEMSLR_ERR_INVALID_ARG;
  if (!c->ready) return fail(c, GEMSLR_ERR_STATE, "halo_plan before setup");
  auto go = [&](const auto &pl) -> gemslr_status {
    if (which > 0 && (level < 0 || level >= pl.st.L)) return GEMSLR_ERR_INVALID_ARG;
    const HaloPlan &h = which == 0 ? pl.hA : (which == 1 ? pl.hE[level] : pl.hF[level]);
    for (int r = 0; r < 2 * pl.nranks; ++r) counts[r] = 0;
    for (size_t i = 0; i < h.peer.size(); ++i) {
      counts[h.peer[i]] = h.soff[i + 1] - h.soff[i];
      counts[pl.nranks + h.peer[i]] = h.roff[i + 1] - h.roff[i];
    }
    if (sglob) std::copy(h.sglob.begin(), h.sglob.end(), sglob);
    if (rglob) std::copy(h.rglob.begin(), h.rglob.end(), rglob);
    return GEMSLR_OK;
  };
  return c->dtype == GEMSLR_F64 ? go(c->ed->plan) : go(c->ez->plan);
}

static gemslr_status need_device(const gemslr_ctx *c) {
  if (!c) return GEMSLR_ERR_INVALID_ARG;
  if (!c->ready) return fail(c, GEMSLR_ERR_STATE, "call before setup");
  if (c->host_only) return fail(c, GEMSLR_ERR_STATE, "host-only context has no device path");
  return GEMSLR_OK;
}

gemslr_status gemslr_spmv(gemslr_ctx *c, const void *x, void *y) {
  gemslr_status st = need_device(c);
  if (st) return st;
  if (!x || !y || x == y) return fail(c, GEMSLR_ERR_INVALID_ARG, "null or aliased vectors");
  return guarded(c, [&]() -> gemslr_status {
    if (c->dtype == GEMSLR_F64) c->ed->spmv((const double *)x, (double *)y, 0, nullptr, nullptr);
    else c->ez->spmv((const cd *)x, (cd *)y, 0, nullptr, nullptr);
    return GEMSLR_OK;
  });
}

gemslr_status gemslr_apply_precond(gemslr_ctx *c, const void *x, void *y) {
  gemslr_status st = need_device(c);
  if (st) return st;
  if (!x || !y || x == y) return fail(c, GEMSLR_ERR_INVALID_ARG, "null or aliased vectors");
  return guarded(c, [&]() -> gemslr_status {
    if (c->dtype == GEMSLR_F64) c->ed->apply_from(0, (const double *)x, (double *)y, nullptr);
    else c->ez->apply_from(0, (const cd *)x, (cd *)y, nullptr);
    return GEMSLR_OK;
  });
}

}  // extern "C"

template <typename T>
static gemslr_status multi_call(gemslr_ctx *c, Engine<T> &E, int which, const void *x, void *y, int nrhs, int64_t ld) {
  using D = typename Dev<T>::type;
  if (nrhs < 1 || ld < E.n) return fail(c, GEMSLR_ERR_INVALID_ARG, "nrhs < 1 or ld < n_local");
  const D *xi = static_cast<const D *>(x);
  D *yo = static_cast<D *>(y);
  if (which == 0 && E.dist) {                                     // several ranks: column by column (halo exchanges)
    for (int q = 0; q < nrhs; ++q) E.spmv(xi + (size_t)q * ld, yo + (size_t)q * ld, 0, nullptr, nullptr);
  } else if (which == 0) {
    E.spmv_multi(xi, yo, ld, nrhs);
  } else if (E.multi_ok()) {
    for (int c0 = 0; c0 < nrhs; c0 += GEMSLR_MAX_RHS)
      E.apply_multi(xi + (size_t)c0 * ld, yo + (size_t)c0 * ld, ld, std::min(GEMSLR_MAX_RHS, nrhs - c0));
  } else {                                                         // kernels without a column dimension
    for (int q = 0; q < nrhs; ++q) E.apply_from(0, xi + (size_t)q * ld, yo + (size_t)q * ld, nullptr);
  }
  return GEMSLR_OK;
}

extern "C" {

gemslr_status gemslr_spmv_multi(gemslr_ctx *c, const void *x, void *y, int nrhs, int64_t ld) {
  gemslr_status st = need_device(c);
  if (st) return st;
  if (!x || !y || x == y) return fail(c, GEMSLR_ERR_INVALID_ARG, "null or aliased blocks");
  return guarded(c, [&]() -> gemslr_status {
    return c->dtype == GEMSLR_F64 ? multi_call(c, *c->ed, 0, x, y, nrhs, ld) : multi_call(c, *c->ez, 0, x, y, nrhs, ld);
  });
}

gemslr_status gemslr_apply_precond_multi(gemslr_ctx *c, const void *x, void *y, int nrhs, int64_t ld) {
  gemslr_status st = need_device(c);
  if (st) return st;
  if (!x || !y || x == y) return fail(c, GEMSLR_ERR_INVALID_ARG, "null or aliased blocks");
  return guarded(c, [&]() -> gemslr_status {
    return c->dtype == GEMSLR_F64 ? multi_call(c, *c->ed, 1, x, y, nrhs, ld) : multi_call(c, *c->ez, 1, x, y, nrhs, ld);
  });
}

gemslr_status gemslr_solve(gemslr_ctx *c, const void *b, void *x, double rtol, int restart, int maxit, int *its,
                           double *hist, int hcap, int *hlen, double *frel) {
  gemslr_status st = need_device(c);
  if (st) return st;
  if (!b || !x || b == x || rtol <= 0 || restart < 1 || maxit < 1 || (hist && hcap < 0))
    return fail(c, GEMSLR_ERR_INVALID_ARG, "bad solve arguments");
  return guarded(c, [&]() -> gemslr_status {
    if (c->dtype == GEMSLR_F64)
      return (gemslr_status)c->ed->solve((const double *)b, (double *)x, rtol, restart, maxit, its, hist, hcap, hlen, frel);
    return (gemslr_status)c->ez->solve((const cd *)b, (cd *)x, rtol, restart, maxit, its, hist, hcap, hlen, frel);
  });
}

}  // extern "C"

template <typename T>
static gemslr_status host_solve(gemslr_ctx *c, Engine<T> &E, const void *b_host, void *x_host, double rtol, int restart,
                                int maxit, int *its, double *hist, int hcap, int *hlen, double *frel) {
  using D = typename Dev<T>::type;
  const int64_t n = E.n, ng = E.nglob;            // local rows, global rows
  cudaStream_t s = c->stream;
  if (!E.xb) {
    E.xb = c->pool.get<D>(2 * (n + 1) + 2 * (ng + 1));
    E.bb = E.xb + (n + 1);
  }
  D *bn = E.bb + (n + 1), *xn = bn + (ng + 1);
  CK(cudaMemcpyAsync(bn, b_host, ng * sizeof(D), cudaMemcpyHostToDevice, s));
  if (x_host) CK(cudaMemcpyAsync(xn, x_host, ng * sizeof(D), cudaMemcpyHostToDevice, s));
  else CK(cudaMemsetAsync(xn, 0, ng * sizeof(D), s));
  const int grid = grid_for((n + 255) / 256, 4);
  k_perm<D><<<grid, 256, 0, s>>>(n, E.perm_d, bn, E.bb, 0);
  k_perm<D><<<grid, 256, 0, s>>>(n, E.perm_d, xn, E.xb, 0);
  int rc = E.solve(E.bb, E.xb, rtol, restart, maxit, its, hist, hcap, hlen, frel);
  k_perm<D><<<grid, 256, 0, s>>>(n, E.perm_d, E.xb, xn, 1);   // owned entries; the others keep x0
  CK(cudaMemcpyAsync(x_host, xn, ng * sizeof(D), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  return (gemslr_status)rc;
}

extern "C" {


gemslr_status gemslr_solve_host(gemslr_ctx *c, const void *b, void *x, double rtol, int restart, int maxit, int *its,
                                double *hist, int hcap, int *hlen, double *frel) {
  gemslr_status st = need_device(c);
  if (st) return st;
  if (!b || !x || rtol <= 0 || restart < 1 || maxit < 1) return fail(c, GEMSLR_ERR_INVALID_ARG, "bad solve arguments");
  return guarded(c, [&]() -> gemslr_status {
    if (c->dtype == GEMSLR_F64) return host_solve(c, *c->ed, b, x, rtol, restart, maxit, its, hist, hcap, hlen, frel);
    return host_solve(c, *c->ez, b, x, rtol, restart, maxit, its, hist, hcap, hlen, frel);
  });
}

static gemslr_status permute_call(gemslr_ctx *c, const void *in, void *out, int inverse) {
  gemslr_status st = need_device(c);
  if (st) return st;
  if (!in || !out || in == out) return fail(c, GEMSLR_ERR_INVALID_ARG, "null or aliased vectors");
  return guarded(c, [&]() -> gemslr_status {
    if (c->dtype == GEMSLR_F64) {
      auto &E = *c->ed;
      k_perm<double><<<grid_for((E.n + 255) / 256, 4), 256, 0, c->stream>>>(E.n, E.perm_d, (const double *)in, (double *)out, inverse);
    } else {
      auto &E = *c->ez;
      k_perm<cd><<<grid_for((E.n + 255) / 256, 4), 256, 0, c->stream>>>(E.n, E.perm_d, (const cd *)in, (cd *)out, inverse);
    }
    CK(cudaGetLastError());
    return GEMSLR_OK;
  });
}

gemslr_status gemslr_to_local(gemslr_ctx *c, const void *xn, void *xl) { return permute_call(c, xn, xl, 0); }
gemslr_status gemslr_to_natural(gemslr_ctx *c, const void *xl, void *xn) { return permute_call(c, xl, xn, 1); }

gemslr_status gemslr_export_setup(const gemslr_ctx *c, const char *dir) {
  if (!c || !dir) return GEMSLR_ERR_INVALID_ARG;
  if (!c->ready) return fail(c, GEMSLR_ERR_STATE, "export before setup");
  return guarded(const_cast<gemslr_ctx *>(c), [&]() -> gemslr_status {
    if (c->dtype == GEMSLR_F64) c->ed->export_bundle(dir); else c->ez->export_bundle(dir);
    return GEMSLR_OK;
  });
}

gemslr_status gemslr_stats(const gemslr_ctx *c, char *json, size_t cap) {
  if (!c || !json || cap == 0) return GEMSLR_ERR_INVALID_ARG;
  if (!c->ready) return fail(c, GEMSLR_ERR_STATE, "stats before setup");
  auto *cc = const_cast<gemslr_ctx *>(c);
  if (cc->prof.on) cc->prof.flush();
  std::string j = c->dtype == GEMSLR_F64 ? c->ed->stats_json() : c->ez->stats_json();
  std::snprintf(json, cap, "%s", j.c_str());
  return j.size() + 1 > cap ? GEMSLR_ERR_INVALID_ARG : GEMSLR_OK;
}

// Debug hook (not in gemslr.h): record a clock64 trace of block 0 of the down-sweep
// trisolve launches into a device buffer of 4 * 4096 int64.
extern "C" void gemslr_debug_trace(void *dev_buf) { g_tri_dbg = static_cast<long long *>(dev_buf); }
extern "C" void gemslr_debug_trace_level(int level) { g_tri_dbg_level = level; }

gemslr_status gemslr_set_orthogonalization(gemslr_ctx *c, int orth) {
  if (!c || orth < 0 || orth > 1) return fail(c, GEMSLR_ERR_INVALID_ARG, "orth must be 0 (CGS2) or 1 (DCGS2)");
  c->orth = orth;
  return GEMSLR_OK;
}

gemslr_status gemslr_profile(gemslr_ctx *c, int enable, int reset) {
  if (!c) return GEMSLR_ERR_INVALID_ARG;
  if (reset) c->prof.reset();
  c->prof.on = enable != 0;
  if (!c->prof.on) c->prof.flush();
  return GEMSLR_OK;
}

const char *gemslr_last_error(const gemslr_ctx *c) { return c ? c->err.c_str() : "null context"; }

void gemslr_destroy(gemslr_ctx *c) {
  if (!c) return;
  if (c->device >= 0) {
    cudaSetDevice(c->device);
    cudaStreamSynchronize(c->stream);
  }
  c->prof.flush();
  c->ed.reset();
  c->ez.reset();
  c->pool.clear();
  delete c;
}

}  // extern "C"
