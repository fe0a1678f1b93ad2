/*
 * gemslr.h — C-ABI of the B200-native GeMSLR solve path (libgemslr.so).
 *
 * Method: parGeMSLR, arXiv 2205.03224 (/root/reference/PAPER.md, cited "P:Lx").
 * The hot path is one preconditioned FGMRES iteration: a CSR SpMV
 * (Note N P:L58-66), one application of the multilevel Schur-complement
 * low-rank preconditioner (Alg. 2) and the Gram-Schmidt dots and
 * norms.  Everything on that path runs in this
 * library's sm_100a kernels; there is no CPU fallback.
 *
 * Conventions (all functions):
 *  - Every entry point returns gemslr_status (0 = OK, >0 = warning, <0 = error)
 *    except gemslr_last_error / gemslr_destroy.  After an error the context
 *    stays usable for a new call; gemslr_last_error() gives a message.
 *  - Collective: with a communicator (nranks > 1) every rank makes the same
 *    sequence of calls.
 *  - Ownership: every input is borrowed.  setup() copies A.  Device buffers
 *    passed to spmv / apply_precond / solve belong to the caller and must not
 *    alias each other.  The context owns factors, low-rank bases, Krylov
 *    workspace and every temporary.
 *  - Vectors on the device are in the LOCAL PERMUTED LAYOUT (gemslr_layout
 *    gives the original row of each local row); scalars are double (GEMSLR_F64)
 *    or interleaved (re, im) double pairs (GEMSLR_C128).
 *  - Streams: work is enqueued on the stream given to gemslr_create (0 = the
 *    legacy default stream).  spmv / apply_precond are asynchronous; solve
 *    returns after completion because it must report the iteration count.
 */
#ifndef GEMSLR_H
#define GEMSLR_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  GEMSLR_OK = 0,
  GEMSLR_NOT_CONVERGED = 1,     /* solve hit maxit; x, its, history still valid (flag F)        */
  GEMSLR_ERR_INVALID_ARG = -1,  /* null pointer, n <= 0, levels < 1, p < 1, rank < 0, restart < 1, rtol <= 0, aliasing */
  GEMSLR_ERR_BAD_CSR = -2,      /* non-monotone rowptr, column out of range, unsorted/duplicate columns        */
  GEMSLR_ERR_PARTITION = -3,    /* p larger than the level-0 vertex count                                      */
  GEMSLR_ERR_ZERO_PIVOT = -4,   /* ILU breakdown; last_error names level, block and row                        */
  GEMSLR_ERR_LOWRANK = -5,      /* |1 - gamma| < 1e-12 among the selected Ritz values, or Arnoldi start = 0    */
  GEMSLR_ERR_STATE = -6,        /* call before setup, setup twice, compute call on a host-only context         */
  GEMSLR_ERR_CUDA = -7,
  GEMSLR_ERR_NCCL = -8,
  GEMSLR_ERR_OOM = -9
} gemslr_status;

typedef enum { GEMSLR_F64 = 0, GEMSLR_C128 = 1 } gemslr_dtype;
typedef enum { GEMSLR_ILU0 = 0, GEMSLR_ILUT = 1 } gemslr_ilu;

/* Setup parameters.  setup(A, levels, k, rank) of the north star reads k as
 * the number of subdomains per level p and rank as the low-rank k (reading
 * Q31 of DESIGN.md). */
typedef struct {
  int levels;               /* l_ev >= 1: number of partition levels                          */
  int subdomains;           /* p >= 1 per level, fixed at every level                         */
  int rank;                 /* low-rank k >= 0, same at every level                    */
  int ilu;                  /* gemslr_ilu: ILU(0) or ILUT for every diagonal block    */
  double ilut_drop;         /* ILUT tau (relative to the row 2-norm; reading Q9)                            */
  int ilut_fill;            /* ILUT lfil: off-diagonals kept per row in each of L and U (reading Q9)        */
  int last_blocks;          /* block-Jacobi blocks of C_{l_ev-1}; 0 = subdomains               */
  double arnoldi_tol;       /* relative change of the selected Ritz values between cycles; 0 = 1e-2 */
  int arnoldi_max_cycles;   /* thick-restart cycles (cycle length m = 2k); 0 = 10                   */
  unsigned long long seed;  /* Arnoldi start vector seed                                                    */
  int cluster_ctas;         /* CTAs per thread-block cluster in the triangular solves; 0 = automatic        */
  int tri_kernel;           /* triangular-solve kernel: 0 = automatic (register-prefetched k_tri_reg where
                               the setup proves it applies), 1 = TMA-staged k_tri_pipe, 2 = level kernel     */
  int root_inner_its;       /* NEXT-1: steps of right-preconditioned GMRES on the root Schur complement
                               S_0 = C_0 - E_0 U_0^-1 L_0^-1 F_0 inside every apply (Alg. 2 line 6, P:L541-545;
                               the experiments use 3 to 5); 0 = the single-pass low-rank branch
                               (reading Q2).  The preconditioner is then nonlinear (use FGMRES).  One GPU. */
  double ilu_shift;         /* complex diagonal shift of the block ILUs: sigma = i*ilu_shift*sum|a_ii|/n added
                               to every B_l and C_last block before factoring (the paper uses
                               0.05); 0 = off; GEMSLR_C128 only (INVALID_ARG for GEMSLR_F64)               */
  int tri_split;            /* CTAs (one thread-block cluster) per subdomain block in the register-prefetched
                               triangular solves: the block's rows cut into that many contiguous chunks on as
                               many SMs, values crossing chunks moved through distributed shared memory; 0 =
                               automatic (the deep level-0 blocks: 4 or 2 when blocks x Q fit the SMs), 1 = off,
                               2 or 4 = forced on every level stage.  The solves compute the same Alg. 2
                               substitutions in the same order inside every row.          */
} gemslr_params;

typedef struct gemslr_ctx gemslr_ctx;

/* Create a context on CUDA device `cuda_device` (>= 0).  cuda_device = -1
 * creates a HOST-ONLY planning context: setup() then runs the host stage
 * (partition, permutation, ILU, schedules) and skips everything that needs the
 * GPU (upload, low-rank Arnoldi); spmv / apply_precond / solve return
 * GEMSLR_ERR_STATE.  It exists so the host logic can be inspected and tested
 * without a GPU.  nccl_comm: ncclComm_t or NULL (single GPU).  cuda_stream:
 * cudaStream_t or NULL (legacy default stream). */
gemslr_status gemslr_create(gemslr_ctx **out, int cuda_device, void *nccl_comm, void *cuda_stream);

/* Multi-GPU (one process per GPU).  gemslr_nccl_unique_id: rank 0
 * creates an NCCL unique id (128 bytes) that the caller broadcasts (e.g. with
 * torch.distributed); nccl_lib = path of libnccl.so.2 to load (NULL: the one
 * already loaded in the process).  gemslr_create_dist: like gemslr_create for
 * rank `rank` of `nranks`; the library owns an NCCL communicator built from
 * nccl_id.  cuda_device = -1 gives a host-only planning context of that rank
 * (no NCCL; used to test ownership and halo plans without GPUs).  With
 * nranks > 1 the matrix is row-partitioned by subdomain: level-0 parts in
 * contiguous rank ranges (p must be a multiple of nranks), later parts
 * and C_last rows to the rank owning most of their earlier-level neighbours;
 * exterior values move by grouped ncclSend/ncclRecv, W^H products, Gram-Schmidt
 * dots and the last separator by ncclAllReduce; the last-separator solve is
 * replicated.  nranks = 1 with a non-NULL nccl_id builds a one-rank
 * NCCL communicator and runs the DISTRIBUTED code path on one GPU (every
 * all-reduce an NCCL call, no halo peers): a check of the NCCL plumbing and of the
 * distributed kernels without a second GPU. */
gemslr_status gemslr_nccl_unique_id(const char *nccl_lib, void *id128);
gemslr_status gemslr_create_dist(gemslr_ctx **out, int cuda_device, void *cuda_stream, int nranks, int rank,
                                 const void *nccl_id, const char *nccl_lib);

/* Host-staged communication backend: the caller supplies the collectives as
 * callbacks on HOST buffers (e.g. torch.distributed over gloo); the library
 * synchronises its stream and stages device data through pinned memory.  It
 * runs the same distributed algorithm as the NCCL backend and lets several
 * ranks share one GPU (each rank only waits on the host, never in a kernel).
 * allreduce: sum `count` doubles in place over all ranks.  sendrecv: for each
 * of the npeers peers send sendcounts[i] doubles and receive recvcounts[i]
 * doubles (a grouped, deadlock-free exchange).  Callbacks return 0 on success. */
typedef int (*gemslr_allreduce_fn)(void *user, double *buf, size_t count);
typedef int (*gemslr_sendrecv_fn)(void *user, int npeers, const int *peers, const double *const *sendbufs,
                                  const size_t *sendcounts, double *const *recvbufs, const size_t *recvcounts);
gemslr_status gemslr_create_hostcomm(gemslr_ctx **out, int cuda_device, void *cuda_stream, int nranks, int rank,
                                     gemslr_allreduce_fn allreduce, gemslr_sendrecv_fn sendrecv, void *user);

/* Halo plan of this rank (inspection/tests): which = 0 SpMV, 1 E_l, 2 F_l (level
 * `level`).  counts (host, 2*nranks): values sent to / received from each rank;
 * sglob, rglob (host, may be NULL): global permuted positions of the values,
 * concatenated by peer in rank order. */
gemslr_status gemslr_halo_plan(const gemslr_ctx *ctx, int which, int level, int64_t *counts, int64_t *sglob,
                               int64_t *rglob);

/* Optional device allocator (e.g. torch's caching allocator).  NULL resets to cudaMalloc/cudaFree. */
gemslr_status gemslr_set_allocator(gemslr_ctx *ctx, void *(*alloc_fn)(size_t bytes, void *user),
                                   void (*free_fn)(void *ptr, void *user), void *user);

/* Optional vertex coordinates (host, n x dim, row-major, copied) for the
 * recursive coordinate bisection partitioner; without them setup() bisects by
 * BFS level sets of |A|+|A^T| (reading Q23).  Call before setup. */
gemslr_status gemslr_set_coordinates(gemslr_ctx *ctx, int dim, const double *coords);

/* setup(A, levels, p, rank) — Alg. 1 pGeMSLRSetup with Alg. 3
 * reordering.  A is the global n x n CSR on the HOST, identical on
 * every rank: rowptr int64[n+1], colidx int32[nnz] (sorted, unique per row),
 * values double[nnz] or (re,im) double[2 nnz].  A is copied; the caller keeps
 * ownership.  Partition, permutation, ILU factors and level schedules are built
 * on the host; the low-rank bases W_l, G_l = (I - R_l)^{-1} - I are built
 * bottom-up by a thick-restart Arnoldi on the GPU using the same
 * kernels as the solve path.  Errors: INVALID_ARG, BAD_CSR, PARTITION,
 * ZERO_PIVOT, LOWRANK, CUDA, OOM, STATE (setup twice). */
gemslr_status gemslr_setup(gemslr_ctx *ctx, gemslr_dtype dtype, int64_t n, const int64_t *rowptr,
                           const int32_t *colidx, const void *values, const gemslr_params *params);

/* Local layout: n_local rows on this rank; global_row_of_local[i] (host,
 * caller-allocated, may be NULL) = original (natural) row of local row i. */
gemslr_status gemslr_layout(const gemslr_ctx *ctx, int64_t *n_local, int64_t *global_row_of_local);

/* y = A x (Note N P:L58-61): diagonal block + off-diagonal block over the halo.
 * x_dev, y_dev: device, n_local scalars, local permuted layout, x != y. */
gemslr_status gemslr_spmv(gemslr_ctx *ctx, const void *x_dev, void *y_dev);

/* y = M^{-1} x: one single-pass application of Alg. 2 (reading Q2),
 * down sweep (ILU solves, E_l coupling, W_l G_l W_l^H correction), bottom
 * block-Jacobi solve of C_{l_ev-1}, up sweep (F_l coupling, ILU
 * solves).  Device pointers, local permuted layout, x != y. */
gemslr_status gemslr_apply_precond(gemslr_ctx *ctx, const void *x_dev, void *y_dev);

/* Several right-hand sides (NEXT-4; the paper's GPU motivation, P:L1285-1286,
 * P:L1326-1330).  x_dev, y_dev: device, column-major n_local x nrhs blocks with
 * leading dimension ld >= n_local (column c at x_dev + c*ld scalars), local
 * permuted layout, x != y.  Results equal nrhs calls of the single-vector
 * function (up to summation order).  The SpMV reads A once for all columns; the
 * apply runs the triangular solves of up to GEMSLR_MAX_RHS columns in one
 * launch per stage (the columns share the factor stream), the E/W coupling per
 * column.  With several ranks (collective) the columns go one by one through the
 * distributed spmv / apply; INVALID_ARG for nrhs < 1 or ld < n_local. */
#define GEMSLR_MAX_RHS 8
gemslr_status gemslr_spmv_multi(gemslr_ctx *ctx, const void *x_dev, void *y_dev, int nrhs, int64_t ld);
gemslr_status gemslr_apply_precond_multi(gemslr_ctx *ctx, const void *x_dev, void *y_dev, int nrhs, int64_t ld);

/* solve(b, x0, tol, restart) -> (x, iterations, residual history): right-
 * preconditioned FGMRES(restart) with CGS2, or DCGS2 after
 * gemslr_set_orthogonalization(ctx, 1) (DESIGN.md readings
 * Q14/Q15/Q38).  b_dev: device, local permuted layout; x_dev: in x0, out x.
 * res_hist (host, may be NULL): relative residual estimates |g_{j+1}|/||b||,
 * entry 0 = initial; *hist_len = number written (<= hist_cap).
 * final_true_relres (may be NULL): ||b - A x||/||b|| recomputed explicitly.
 * Returns GEMSLR_NOT_CONVERGED if maxit was reached. */
gemslr_status gemslr_solve(gemslr_ctx *ctx, const void *b_dev, void *x_dev, double rtol, int restart,
                           int maxit, int *iterations, double *res_hist, int hist_cap, int *hist_len,
                           double *final_true_relres);

/* Orthogonalisation of the solves that follow on this context (default 0):
 * 0 = CGS2 (DESIGN.md c5, reading Q14): classical Gram-Schmidt applied twice at
 *     every step, three passes over the Krylov basis;
 * 1 = DCGS2 (c5', reading Q38): the same two projections with the second one and
 *     the normalisation delayed to the next step, where they share its passes
 *     (one dot pass + one update pass per step); z_j = M(u_j) of the not yet
 *     normalised u_j, which flexible GMRES admits.
 * Any other value: GEMSLR_ERR_INVALID_ARG.  No GPU work; the context keeps it. */
gemslr_status gemslr_set_orthogonalization(gemslr_ctx *ctx, int orth);

/* The same solve with HOST vectors in the ORIGINAL (natural) global order,
 * length n (global): the host->device copy, the permutation into the local
 * layout, the solve, the inverse permutation and the device->host copy all
 * happen inside the call (the end-to-end path).  x_host: in x0, out x; with
 * nranks > 1 only the entries this rank owns are written. */
gemslr_status gemslr_solve_host(gemslr_ctx *ctx, const void *b_host, void *x_host, double rtol, int restart,
                                int maxit, int *iterations, double *res_hist, int hist_cap, int *hist_len,
                                double *final_true_relres);

/* Natural <-> local permuted layout on the device (kernel K14). */
gemslr_status gemslr_to_local(gemslr_ctx *ctx, const void *x_natural_dev, void *x_local_dev);
gemslr_status gemslr_to_natural(gemslr_ctx *ctx, const void *x_local_dev, void *x_natural_dev);

/* Write the setup bundle (manifest.json + raw little-endian .bin arrays) to
 * directory `dir` (created if missing): permutation, level / block offsets,
 * every ILU factor (block-local CSR), W_l (s_l x k_l column-major, rows in the
 * global permuted order of J_l), R_l, G_l.  This is what tests/ hand to the
 * independent oracle verifier.  Collective with several ranks: the rows of W_l are
 * gathered (one all-reduce per level), rank 0 writes the bundle, and
 * the factors are omitted (each rank holds only its own blocks; the oracle
 * recomputes all of them from its own A). */
gemslr_status gemslr_export_setup(const gemslr_ctx *ctx, const char *dir);

/* JSON statistics: levels achieved, level offsets, block counts, nnz of the
 * factors (fill), triangular-solve depths, ranks, Arnoldi cycles, per-kernel
 * timing (when enabled), collective counts. */
gemslr_status gemslr_stats(const gemslr_ctx *ctx, char *json, size_t cap);

/* Per-kernel CUDA-event timing on the context stream (bench roofline):
 * enable != 0 records an event pair around every launch; reset clears the sums. */
gemslr_status gemslr_profile(gemslr_ctx *ctx, int enable, int reset);

const char *gemslr_last_error(const gemslr_ctx *ctx);
void gemslr_destroy(gemslr_ctx *ctx);

#ifdef __cplusplus
}
#endif
#endif /* GEMSLR_H */
