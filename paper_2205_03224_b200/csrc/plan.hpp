// Host-side setup data of the GeMSLR solve path (arXiv 2205.03224).
//
// The host setup (partition -> multilevel permutation -> blocks -> ILU ->
// level schedules) produces a HostPlan; context.cu uploads it and builds the
// low-rank terms on the GPU.  Notation follows the paper: level l has the
// interiors I_l = [o_l, o_{l+1}) split into p subdomain blocks B_l^(j), the
// interface below it J_l = [o_{l+1}, N), and the last separator
// C_{l_ev-1} = [o_L, N).
#pragma once

#include <complex>
#include <cstdint>
#include <string>
#include <vector>

namespace gemslr {

using zc = std::complex<double>;

inline double absval(double a) { return a < 0 ? -a : a; }
inline double absval(const zc &a) { return std::abs(a); }
inline double abs2(double a) { return a * a; }
inline double abs2(const zc &a) { return a.real() * a.real() + a.imag() * a.imag(); }

struct Error {
  int code;
  std::string msg;
};

// Symmetric adjacency graph of |A| + |A^T| without self loops.
struct Graph {
  int64_t n = 0;
  std::vector<int64_t> ptr;
  std::vector<int32_t> adj;
};

// Multilevel structure (Alg. 3).  Positions are in the global
// permuted order Â = Pᵀ A P with perm[new] = old.
struct Structure {
  int64_t n = 0;
  int L = 0;                                   // achieved levels l_ev
  std::vector<int64_t> perm, iperm;
  std::vector<int64_t> o;                      // o_0 .. o_L
  std::vector<std::vector<int64_t>> blk;       // per level: block boundaries (absolute)
  std::vector<int64_t> last;                   // C_last block boundaries (absolute)
};

template <typename T>
struct Csr {                                    // rows local to a range, columns as documented per use
  int64_t n = 0, m = 0;
  std::vector<int64_t> ptr;
  std::vector<int32_t> col;
  std::vector<T> val;
  int64_t nnz() const { return ptr.empty() ? 0 : ptr[n]; }
};

// ILU factors of one diagonal block in block-local indices: L strictly lower
// with an implicit unit diagonal, U upper with the diagonal FIRST in each row.
template <typename T>
struct Factor {
  Csr<T> L, U;
};

// Level-scheduled, SELL-32 packed triangular sweep over a set of blocks
// ("stage").  For block b, levels [blk_lev[b], blk_lev[b+1]) of lev_slice;
// level v covers slices [lev_slice[v], lev_slice[v+1]); slice s has 32 lanes
// (one row each, -1 = padding) and width w_s = (slice_off[s+1]-slice_off[s])/32
// entries stored column-major (entry e of lane r at slice_off[s] + 32 e + r).
// Rows and columns are ABSOLUTE positions in the permuted vector; col = -1 pads.
template <typename T>
struct TriPack {
  std::vector<int32_t> blk_lev;
  std::vector<int32_t> lev_slice;
  std::vector<int64_t> slice_off;
  std::vector<int32_t> slice_row;
  std::vector<int32_t> col;
  std::vector<T> val;
  std::vector<T> diag;                          // U sweep only: u_ii per lane (1 on padding)
  int max_depth = 0;
  int64_t nnz_real = 0;                         // stored nonzeros without padding
};

// TMA-pipelined form of a stage's two sweeps (k_tri_pipe): per block, the L
// chunks then the U chunks; a chunk is <= PIPE_NW slices of ONE level whose
// static data is one contiguous, 128-byte aligned blob of <= PIPE_SB bytes:
//   int32 header: ns, s0 (block-relative first slice), ne, flags (bit0 = U
//     sweep), ns + 1 relative entry offsets, padded to 16 bytes;
//   int32 rows[ns*32]; int32 aux[ns*32] (L chunks: packed U index of the row);
//   T diag[ns*32] (U sweep: 1/u_ii; 1 in L chunks); int32 col[ne]; T val[ne].
// The right-hand sides of a chunk are contiguous in a packed per-sweep vector
// (index = stage slice * 32 + lane) and arrive by a second bulk copy.
// Column encoding: c >= 0 block-relative position (slice * 32 + lane) of the
// dependency, read from the shared-memory ring of the last `ring` solution
// values; c == -1 padding; c <= -2 "far" dependency read from global memory
// at row -c - 2.
struct ChunkDesc {                          // 16 bytes, one vector load in the producer
  int32_t blob128;                          // blob offset / 128
  int32_t bytes;                            // blob bytes
  int32_t slice;                            // first stage slice (packed right-hand sides at slice * 32)
  int32_t nsflags;                          // ns << 1 | (1 if U sweep)
};
constexpr int PIPE_NW = 8;                  // consumer warps per CTA = max slices per chunk
constexpr int PIPE_SB = 30 * 1024;          // blob bytes per pipeline stage
constexpr int PIPE_RING_ENTRIES = 16384;     // solution window (double; 8192 for complex)

template <typename T>
struct PipePack {
  bool ok = false;
  int ring = 0;                             // entries (power of two)
  std::vector<uint8_t> blob;
  std::vector<ChunkDesc> chunks;
  std::vector<int32_t> blk_chunk;           // per block: [blk_chunk[b], blk_chunk[b+1])
  std::vector<int32_t> blk_nl;              // per block: number of L chunks
  std::vector<int32_t> lpos;                // per stage row: packed L index
  int64_t lslices = 0, uslices = 0;
  int64_t near = 0, far = 0;
};

// Register-prefetched form of a stage's two sweeps (k_tri_reg).  Per block and
// sweep the slices are numbered in level order; slice s goes to consumer warp
// s mod NW, which loads its record straight into registers two slices ahead.
// Records have ONE size per stage (W = reg_width(widest slice) entries), so a
// record's address is plain arithmetic on the slice index — no loaded header
// feeds an address (a loaded address would make the warp wait on the load
// before it reaches the next level barrier).  Record of a slice, 128-byte
// aligned, for lane r:
//   values and ring slots in 16-byte units per lane, so a warp's load is one
//   512-byte LDG.128: T val[W/VE][32][VE] (VE = 16 / sizeof(T) entries per unit,
//   0 on padding); uint16 col[ceil(W/8)][32][8] ring slots (padding -> slot
//   ring-1); int32 out[32]; T rdiag[32] = 1/u_ii (U sweep; 1 in the L sweep).  The level of every record (uint16 `slev`, in the
//   sweep) is copied to shared memory at kernel start: the barrier count of a
//   warp never waits on a global load.
// out: L sweep -> stage-global packed U position (where the U sweep reads its
// right-hand side), U sweep -> the row; -1 = padding lane.
// binfo per block (REG_BINFO ints): L first record, L slices, L levels, U first
// record, U slices, U levels, first lev_off entry of L, of U, first row, end
// row, stage-global packed L slice of the block's first L slice (right-hand
// sides rhsL[(base + s) * 32 + lane]), same for U (mid).
// lev_off: per block and sweep, the first record of every level and the end.
//
// Split form (Q > 1, the level-0 subdomains when Q x blocks fit the SMs): block b
// is cut into Q contiguous row ranges ("chunks", rows [n q / Q, n (q+1) / Q) of the
// block order), chunk q of block b is "block" b Q + q of the pack and runs on CTA
// q of a Q-CTA cluster.  Levels are those of the whole block's DAG; a chunk keeps
// the levels in which it has rows (its local levels).  Because L is lower and U
// upper triangular in the block order, chunk q's L rows depend only on chunks
// <= q and its U rows only on chunks >= q: with chunks at least one dependency
// bandwidth thick, only on q - 1 (L) and q + 1 (U).  Those values ("imports")
// arrive by asynchronous DSMEM stores (st.async) from the producing CTA into an
// import area after the ring (slots R + i: L imports, R + IL + i: U imports), each
// completing its bytes on the consumer's mbarrier of the producer's local level;
// the consumer's slice waits on the barriers of the producer levels it needs
// (sneed).  The producer never waits for the consumer, so the CTAs of a block
// run pipelined one hand-off apart instead of paying it per level.
// Record extension: int32 exp[32] after rdiag (import index in the consumer's
// area of this sweep, -1 none).
// Look-ahead (round 2): with la = REG_LA the last la columns of every record hold the
// entries on the previous level (at most la per row; "new"), the first W - la columns the
// entries on older levels and the imports ("old"; a lane's surplus old entries fill its
// unused new columns).  k_tri_reg sums the old columns after the barrier two levels back,
// while the previous level still runs; after the last barrier only the new columns remain
// on the critical path.  A stage with a row of more than la new entries keeps la = 0.
constexpr int REG_LA = 3;
constexpr int REG_RING_BYTES = 128 * 1024;     // solution window: 16384 doubles / 8192 complex
constexpr int REG_BINFO_INTS = 16;             // + split: producer-L xexp offset, producer-L levels, same for U
inline int reg_width(int w) { return w <= 4 ? 4 : w <= 8 ? 8 : w <= 10 ? 10 : w <= 12 ? 12 : w <= 16 ? 16 : 0; }
template <typename T>
inline size_t reg_record_bytes(int W, bool split = false) {
  const size_t b = (size_t)W * 32 * sizeof(T) + (size_t)((W + 7) / 8) * 32 * 16 + 32 * 4 + 32 * sizeof(T) +
                   (split ? 32 * 4 : 0);
  return (b + 127) / 128 * 128;
}
template <typename T>
struct RegPack {
  bool ok = false;
  int ring = 0;
  int wmax = 0;                                 // widest slice of the stage
  int W = 0;                                    // record width (reg_width(wmax))
  size_t rec_bytes = 0;
  std::vector<uint8_t> data;
  std::vector<uint16_t> slev;                   // per record: level in its sweep
  int max_block_slices = 0;                     // L + U records of the largest block
  std::vector<int32_t> binfo;                   // REG_BINFO_INTS per block
  std::vector<int32_t> lev_off;
  std::vector<int32_t> lpos;                    // per stage row: packed L index
  int64_t lslices = 0, uslices = 0, nrec = 0;
  int64_t near = 0, far = 0;
  int max_levels = 0;
  // split form (Q > 1): import areas (entries, max over chunks), producer level
  // tables, per-record prefix-max of the producer level needed (+1, 0 = none)
  int Q = 1;
  int la = 0;                                   // look-ahead new columns (0 or REG_LA)
  int imp_L = 0, imp_U = 0;                     // IL, IU
  int plev_L = 0, plev_U = 0;                   // max producer local levels (counter / xexp table sizes)
  std::vector<uint16_t> sneed;                  // per record
  std::vector<uint16_t> xexp;                   // per chunk and sweep: values exported per local level
  int64_t exports = 0;
  int nsweep = 2;                               // 2: (L, U); 3: the tail form (binfo layout below)
  bool xmode = false;                           // one-CTA imports: far / cross dependencies at R + i (exp)
  std::vector<int64_t> sw_slices;               // slices of every sweep (stage-global)
};

// Tail form of a stage's sweeps (DESIGN 6b; requires every block's rows adjacent to a
// later level to be its last rows, tails[b] on): with t = L^-1 b1 and ts the tail start,
//   DOWN: L_hh (head rows), L_t|h (tail rows), U_tt (tail rows): t, and z1 on the tail
//         only, which is all E_l reads (Alg. 2 l.3-4);
//   UP:   L_tt on (F_l y2)_tail (u; zero on the head), U_tt and U_h|t on t - [0; u]:
//         y1 = U^-1 (t - L^-1 F_l y2) = z1 - U^-1 L^-1 F_l y2 (Alg. 2 l.9).
// Every one of these sweeps has a shallow DAG (C5 level 0: 337 + 14 + 95 and 14 + 95 +
// 335 levels, against 360 + 456 per full sweep pair); all are exact (rounding only).
// Record binfo layout (3 sweeps): [3k, 3k+1, 3k+2] first record, slices, levels of sweep
// k; [9 + k] its first stage slice.  An entry of a row on a value of the other part
// ("cross": L_t|h's head columns, U_h|t's tail columns) reads a shared-memory slot
// R + i that the producing lane of an earlier sweep wrote (its record's exp field).
// Positions: "Ucat" = [U_tt | U_h|t] packed order (t and u live there), L right-hand
// sides of the DOWN in [L_hh | L_t|h] order.
template <typename T>
struct TailPack {
  bool ok = false;
  std::vector<int64_t> ts;                      // per block: tail start (absolute)
  TriPack<T> Lhh, Lth, Utt, Uht, Ltt;
  RegPack<T> D, U;                              // DOWN (Lhh, Lth, Utt), UP (Ltt, Utt, Uht)
  int32_t nUtt = 0, nLhh = 0;                   // packed entries of U_tt, of L_hh
  std::vector<int32_t> ucat;                    // per stage row: Ucat position
  std::vector<int32_t> lcat;                    // per stage row: DOWN L position ([L_hh | L_t|h])
  std::vector<int32_t> lrow;                    // per DOWN L position: the row (-1 padding)
  std::vector<int32_t> uttpos;                  // per stage row: U_tt position (-1 off the tail)
  std::vector<int32_t> lttpos;                  // per stage row: L_tt position (-1 off the tail)
  int64_t tail_rows = 0;
};

template <typename T>
struct Stage {                                  // the blocks of one level (or of C_last)
  std::vector<int64_t> blk;                     // absolute boundaries (empty blocks removed)
  TriPack<T> Lp, Up;
  PipePack<T> pipe;
  RegPack<T> reg;
  TailPack<T> tail;
};

// Neighbour exchange of one distributed operator: this rank
// sends sidx[soff[i]..soff[i+1]) (local indices) to peer[i] and receives
// roff[i+1]-roff[i] values from peer[i] into its halo buffer at roff[i].
// sglob / rglob are the global permuted positions of those values.
struct HaloPlan {
  std::vector<int32_t> peer;
  std::vector<int64_t> soff{0}, roff{0};
  std::vector<int32_t> sidx;
  std::vector<int64_t> sglob, rglob;
  int64_t nsend() const { return soff.back(); }
  int64_t nrecv() const { return roff.back(); }
};

// Everything below is for THIS rank of `nranks` (one rank: the global problem).
// Local layout: the owned global positions in ascending order, which is
// level-major ([owned I_0 | owned I_1 | ... | owned C_last rows]); lo[l] is the
// local start of level l and lo[L] the start of the owned C_last rows.
// Column conventions of the local operators:
//   Aloc, E_l: c < nloc local, else halo index c - nloc (hA / hE[l]);
//   F_l: c < nloc local, c < nloc + hF[l].nrecv() halo, else the C_last
//        index c - nloc - nrecv of the replicated last-separator vector (nranks > 1).
template <typename T>
struct HostPlan {
  Structure st;
  Csr<T> Ahat;                                  // Pᵀ A P, global, absolute columns
  int nranks = 1, rank = 0;
  std::vector<int32_t> owner;                   // per global position
  std::vector<int64_t> gpos;                    // local -> global position
  std::vector<int64_t> lo;                      // local level offsets (L + 1 entries)
  int64_t nloc = 0, slast = 0;
  Csr<T> Aloc;                                  // owned rows of Â, local columns
  HaloPlan hA;
  std::vector<HaloPlan> hE, hF;
  std::vector<int32_t> last_idx;                // owned C_last rows: index inside C_last
  std::vector<std::vector<Factor<T>>> fac;      // per level, per global block (owned blocks filled)
  std::vector<Factor<T>> lastfac;               // per C_last block (replicated)
  std::vector<Csr<T>> E;                        // E_l: owned rows of J_l (local row - lo[l+1])
  std::vector<Csr<T>> F;                        // F_l: owned rows of I_l (local row - lo[l])
  std::vector<Stage<T>> stage;                  // per level: owned blocks, local rows
  Stage<T> last_stage;                          // all C_last blocks, rows relative to o_L
  int64_t fac_nnz = 0;                          // nnz(L+U) of the factors held by this rank
};

struct SetupOptions {
  int levels = 1, p = 1, ilu = 0, lfil = 10, last_blocks = 0;
  int nranks = 1, rank = 0;
  double tau = 1e-3;
  double shift = 0.0;                           // complex ILU shift factor, complex only
  int coord_dim = 0;
  const double *coords = nullptr;               // n x coord_dim (optional)
  int split = 0;                                // triangular-solve clusters per block: 0 auto, 1 off, 2/4 forced
  int sms = 148;                                // SMs of the device (auto split: blocks x Q must fit)
  int tail = 1;                                 // boundary rows last in each B_l, tail sweeps (DESIGN 6b)
  int tail_dist = 4;                            // tail colouring distance (measured: C5 its 63/64/65/64 at 1-4, fastest at 4)
};

// partition.cpp
Graph build_graph(int64_t n, const int64_t *rowptr, const int32_t *colidx);
bool build_structure(const Graph &g, const SetupOptions &opt, Structure &st, Error &err);

// ilu.cpp
template <typename T> bool ilu0(const Csr<T> &B, Factor<T> &F, std::string &err);
template <typename T> bool ilut(const Csr<T> &B, double tau, int lfil, Factor<T> &F, std::string &err);

// schedule.cpp
template <typename T> void pack_stage(const std::vector<int64_t> &blk, const std::vector<Factor<T>> &fac, Stage<T> &S,
                                      int Q = 1, const std::vector<int64_t> *tails = nullptr);

// hostplan.cpp
template <typename T>
bool build_host_plan(int64_t n, const int64_t *rowptr, const int32_t *colidx, const T *vals,
                     const SetupOptions &opt, HostPlan<T> &plan, Error &err);

// schur.cpp — dense complex Schur machinery for the thick-restart Arnoldi.
// Matrices column-major, leading dimension = rows.
// schur_complex: A (n x n) -> T (upper triangular) and Z (unitary), A = Z T Z^H.
bool schur_complex(int n, const zc *A, zc *T, zc *Z);
// reorder T/Z so that the eigenvalues flagged in `select` come first (in their
// current relative order); Givens swaps of adjacent 1x1 blocks.
void schur_reorder(int n, zc *T, zc *Z, const std::vector<char> &select);

}  // namespace gemslr
