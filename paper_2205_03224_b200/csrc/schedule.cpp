#include <cstdio>
#include <cstdlib>
// Level schedules of the triangular substitutions (built once at setup) and
// their SELL-32 packing for the sm_100a trisolve kernel.
//
// Forward sweep (L, unit diagonal): level(i) = 1 + max level(j), j < i in row i
// of L.  Backward sweep (U): level(i) = 1 + max level(j), j > i in row i of U,
// rows taken in descending order.  Rows of one level are independent; inside a
// level they are sorted ascending and packed 32 per slice (one row per lane),
// entries column-major inside the slice so a warp's loads are coalesced.
#include <algorithm>
#include <chrono>
#include <unordered_map>

#include "plan.hpp"

namespace gemslr {

namespace {

size_t al16_h(size_t b) { return (b + 15) & ~(size_t)15; }

// Q > 1 (split form, plan.hpp RegPack): block b is packed as Q chunks of
// contiguous rows, each with the levels of the whole block's DAG in which it has
// rows; "block" b Q + q of the pack is chunk q of block b.
// Tail sweeps (DESIGN 6b): rsel = 1 keeps the head rows [0, ts_b) of every block, rsel = 2
// the tail rows [ts_b, n_b).  An entry whose column lies in the other part ("cross": its
// value comes from an earlier sweep of the launch) is kept when `cross` is set, else
// dropped (it multiplies a zero); cross entries do not count for the levels.
template <typename T>
void pack_sweep(const std::vector<int64_t> &blk, const std::vector<Factor<T>> &fac, bool upper, TriPack<T> &P,
                int Q = 1, int rsel = 0, const std::vector<int64_t> *ts = nullptr, bool cross = false) {
  P = TriPack<T>();
  P.blk_lev.push_back(0);
  P.lev_slice.push_back(0);
  P.slice_off.push_back(0);
  const size_t nb = fac.size();
  for (size_t b = 0; b < nb; ++b) {
    const Csr<T> &M = upper ? fac[b].U : fac[b].L;
    const int64_t n = M.n;
    const int64_t row0 = blk[b];
    const int64_t tb = rsel ? std::min<int64_t>(std::max<int64_t>((*ts)[b], 0), n) : 0;
    const int64_t i_lo = rsel == 2 ? tb : 0, i_hi = rsel == 1 ? tb : n;   // selected rows (and dependencies)
    auto in_sel = [&](int64_t j) { return j >= i_lo && j < i_hi; };
    std::vector<int32_t> lev(n, 0);
    int32_t nlev = 0;
    if (!upper) {
      for (int64_t i = i_lo; i < i_hi; ++i) {
        int32_t v = 0;
        for (int64_t p = M.ptr[i]; p < M.ptr[i + 1]; ++p)
          if (in_sel(M.col[p])) v = std::max(v, lev[M.col[p]] + 1);
        lev[i] = v;
        nlev = std::max(nlev, v + 1);
      }
    } else {
      for (int64_t i = i_hi - 1; i >= i_lo; --i) {
        int32_t v = 0;
        for (int64_t p = M.ptr[i] + 1; p < M.ptr[i + 1]; ++p)
          if (in_sel(M.col[p])) v = std::max(v, lev[M.col[p]] + 1);
        lev[i] = v;
        nlev = std::max(nlev, v + 1);
      }
    }
    if (i_hi <= i_lo) nlev = 0;
    P.max_depth = std::max(P.max_depth, (int)nlev);
    std::vector<int32_t> ll;                                      // L levels (U packing order inside a level)
    if (upper) {
      const Csr<T> &Lm = fac[b].L;
      ll.assign(n, 0);
      for (int64_t i = 0; i < n; ++i) {
        int32_t v = 0;
        for (int64_t p = Lm.ptr[i]; p < Lm.ptr[i + 1]; ++p) v = std::max(v, ll[Lm.col[p]] + 1);
        ll[i] = v;
      }
    }
   for (int q = 0; q < Q; ++q) {
    const int64_t c0 = n * q / Q, c1 = n * (q + 1) / Q;            // this chunk's rows
    // bucket rows by level (ascending row inside a level)
    std::vector<int64_t> cnt(nlev + 1, 0);
    for (int64_t i = std::max(c0, i_lo); i < std::min(c1, i_hi); ++i) cnt[lev[i] + 1]++;
    for (int32_t v = 0; v < nlev; ++v) cnt[v + 1] += cnt[v];
    std::vector<int64_t> rows(cnt[nlev]);
    {
      std::vector<int64_t> pos(cnt.begin(), cnt.end() - 1);
      for (int64_t i = std::max(c0, i_lo); i < std::min(c1, i_hi); ++i) rows[pos[lev[i]]++] = i;
    }
    if (upper) {
      // Inside a U level, order the rows by their L level (ascending row within
      // it), the order of the L packing: the rows of one L slice that share a U
      // level become adjacent in the U packing, so the L sweep's stores of its
      // results at their U positions coalesce.  Any order inside a level is valid.
      for (int32_t v = 0; v < nlev; ++v)
        std::stable_sort(rows.begin() + cnt[v], rows.begin() + cnt[v + 1],
                         [&](int64_t a, int64_t c) { return ll[a] < ll[c]; });
    }
    auto len = [&](int64_t i) { return M.ptr[i + 1] - M.ptr[i]; };
    (void)len;
    for (int32_t v = 0; v < nlev; ++v) {
      if (Q > 1 && cnt[v + 1] == cnt[v]) continue;                 // a level without rows of this chunk
      for (int64_t s0 = cnt[v]; s0 < cnt[v + 1]; s0 += 32) {
        const int64_t s1 = std::min<int64_t>(s0 + 32, cnt[v + 1]);
        int64_t width = 0;
        for (int64_t t = s0; t < s1; ++t) {
          const int64_t i = rows[t];
          int64_t len = 0;
          for (int64_t p = M.ptr[i] + (upper ? 1 : 0); p < M.ptr[i + 1]; ++p) len += (cross || in_sel(M.col[p])) ? 1 : 0;
          width = std::max(width, len);
        }
        const int64_t off = P.slice_off.back();
        P.col.resize(off + 32 * width, -1);
        P.val.resize(off + 32 * width, T(0));
        for (int lane = 0; lane < 32; ++lane) {
          const int64_t t = s0 + lane;
          if (t >= s1) {
            P.slice_row.push_back(-1);
            if (upper) P.diag.push_back(T(1));
            continue;
          }
          const int64_t i = rows[t];
          P.slice_row.push_back((int32_t)(row0 + i));
          const int64_t pb = M.ptr[i] + (upper ? 1 : 0);
          for (int64_t p = pb, e = 0; p < M.ptr[i + 1]; ++p) {
            if (!cross && !in_sel(M.col[p])) continue;
            P.col[off + 32 * e + lane] = (int32_t)(row0 + M.col[p]);
            P.val[off + 32 * e + lane] = M.val[p];
            P.nnz_real++;
            ++e;
          }
          if (upper) P.diag.push_back(M.val[M.ptr[i]]);
        }
        P.slice_off.push_back(off + 32 * width);
      }
      P.lev_slice.push_back((int32_t)(P.slice_off.size() - 1));
    }
    P.blk_lev.push_back((int32_t)(P.lev_slice.size() - 1));
   }
  }
}

// Chunk the level-scheduled sweeps of every block into TMA blobs (PipePack).
template <typename T>
void pack_pipe(const std::vector<int64_t> &blk, const TriPack<T> &Lp, const TriPack<T> &Up, PipePack<T> &P) {
  P = PipePack<T>();
  P.ring = sizeof(T) == 8 ? PIPE_RING_ENTRIES : PIPE_RING_ENTRIES / 2;
  const int R = P.ring;
  const size_t nb = blk.size() - 1;
  const int64_t R0 = blk.front(), NR = blk.back() - blk.front();
  P.blk_chunk.push_back(0);
  P.lslices = (int64_t)Lp.slice_row.size() / 32;
  P.uslices = (int64_t)Up.slice_row.size() / 32;
  // packed index (slice * 32 + lane, stage-global) of every row in each sweep
  std::vector<int32_t> upos(NR, -1);
  P.lpos.assign(NR, -1);
  for (int64_t s = 0; s < P.lslices; ++s)
    for (int lane = 0; lane < 32; ++lane) {
      const int32_t row = Lp.slice_row[s * 32 + lane];
      if (row >= 0) P.lpos[row - R0] = (int32_t)(s * 32 + lane);
    }
  for (int64_t s = 0; s < P.uslices; ++s)
    for (int lane = 0; lane < 32; ++lane) {
      const int32_t row = Up.slice_row[s * 32 + lane];
      if (row >= 0) upos[row - R0] = (int32_t)(s * 32 + lane);
    }
  auto align = [](size_t v, size_t a) { return (v + a - 1) / a * a; };
  auto blob_bytes = [&](int32_t ns, size_t ne) {
    return align((size_t)(ns + 5), 4) * 4 + (size_t)ns * 32 * 4 * 2 + (size_t)ns * 32 * sizeof(T) + ne * (4 + sizeof(T));
  };
  for (size_t b = 0; b < nb; ++b) {
    int32_t nL = 0;
    for (int sweep = 0; sweep < 2; ++sweep) {
      const TriPack<T> &S = sweep ? Up : Lp;
      const bool upper = sweep == 1;
      const int32_t lv0 = S.blk_lev[b], lv1 = S.blk_lev[b + 1];
      if (lv1 <= lv0) continue;
      const int32_t sb0 = S.lev_slice[lv0];
      // chunk boundaries: <= PIPE_NW slices of one level, blob <= PIPE_SB bytes
      struct Ch { int32_t s0, s1, lev_end; };
      std::vector<Ch> ch;
      for (int32_t v = lv0; v < lv1; ++v) {
        int32_t s = S.lev_slice[v];
        while (s < S.lev_slice[v + 1]) {
          Ch c{s, s, S.lev_slice[v + 1]};
          size_t ne = 0;
          while (c.s1 < S.lev_slice[v + 1] && c.s1 - c.s0 < PIPE_NW) {
            const size_t e2 = ne + (size_t)(S.slice_off[c.s1 + 1] - S.slice_off[c.s1]);
            if (blob_bytes(c.s1 + 1 - c.s0, e2) > (size_t)PIPE_SB) {
              if (c.s1 == c.s0) return;             // one slice does not fit: no pipelined form
              break;
            }
            ne = e2;
            c.s1++;
          }
          ch.push_back(c);
          s = c.s1;
        }
      }
      for (const Ch &c : ch) {
        const int32_t ns = c.s1 - c.s0;
        const int64_t e0 = S.slice_off[c.s0], e1 = S.slice_off[c.s1];
        const int32_t ne = (int32_t)(e1 - e0);
        const size_t H = align((size_t)(ns + 5), 4);
        const size_t bytes = blob_bytes(ns, (size_t)ne);
        const size_t off = align(P.blob.size(), 128);
        P.blob.resize(off + bytes, 0);
        uint8_t *base = P.blob.data() + off;
        int32_t *hdr = reinterpret_cast<int32_t *>(base);
        int32_t *rows = hdr + H;
        int32_t *aux = rows + ns * 32;
        T *diag = reinterpret_cast<T *>(aux + ns * 32);
        int32_t *col = reinterpret_cast<int32_t *>(diag + ns * 32);
        T *val = reinterpret_cast<T *>(col + ne);
        // chunks of one level run without a barrier between them, so a dependency
        // stays in the ring only if no write of the whole level can overwrite it
        const int32_t send = c.lev_end - sb0;         // level end (block-relative slice)
        hdr[0] = ns;
        hdr[1] = c.s0 - sb0;
        hdr[2] = ne;
        hdr[3] = (upper ? 1 : 0) | (c.s1 == c.lev_end ? 2 : 0);
        for (int32_t i = 0; i < ns; ++i) {
          const int32_t s = c.s0 + i;
          hdr[4 + i] = (int32_t)(S.slice_off[s] - e0);
          for (int lane = 0; lane < 32; ++lane) {
            const int32_t row = S.slice_row[(int64_t)s * 32 + lane];
            rows[i * 32 + lane] = row;
            aux[i * 32 + lane] = (!upper && row >= 0) ? upos[row - R0] : -1;
            diag[i * 32 + lane] = upper ? T(1) / S.diag[(int64_t)s * 32 + lane] : T(1);   // reciprocal
          }
          const int w = (int)((S.slice_off[s + 1] - S.slice_off[s]) / 32);
          for (int e = 0; e < w; ++e)
            for (int lane = 0; lane < 32; ++lane) {
              const int64_t g = S.slice_off[s] + 32 * e + lane;
              const int64_t l = g - e0;
              const int32_t dep = S.col[g];
              val[l] = S.val[g];
              if (dep < 0) { col[l] = -1; continue; }
              const int32_t pd = sweep ? upos[dep - R0] : P.lpos[dep - R0];
              const int32_t q = pd - sb0 * 32;          // block-relative position
              if ((int64_t)send * 32 - 1 - q < R) { col[l] = q; P.near++; }
              else { col[l] = -dep - 2; P.far++; }
            }
        }
        hdr[4 + ns] = ne;
        P.chunks.push_back(ChunkDesc{(int32_t)(off / 128), (int32_t)bytes, c.s0, (ns << 1) | (upper ? 1 : 0)});
        if (!upper) nL++;
      }
    }
    P.blk_chunk.push_back((int32_t)P.chunks.size());
    P.blk_nl.push_back(nL);
  }
  P.blob.resize(align(P.blob.size(), 128), 0);
  P.ok = true;
}

// Shared-memory wavefronts of the W gathers of one record.  Column e is one
// LDS.64 (LDS.128 for complex) of 32 lanes, served per half-warp (lanes 0-15,
// 16-31; per quarter for 16-byte slots): a part costs the largest number of
// distinct slots that fall into one of its G = 128 / sizeof(T) bank groups (the
// ncu ideal is 2 wavefronts per LDS.64).  After the greedy order of pack_reg,
// swap a lane's entries between two columns while that lowers the summed cost
// (any entry order of a lane gives the same sum up to rounding).  C5 level 0:
// 3.49 wavefronts per LDS.64 with the whole-warp greedy, 3.21 with the per-part
// greedy, 2.86 after this pass (GEMSLR_DEBUG_BANKS=1 prints it; ideal 2).
// Returns {cost before, cost after}.
template <typename T>
static std::pair<int, int> refine_record(uint8_t *base, int W, int wo) {
  const int VE = 16 / (int)sizeof(T), G = (int)(128 / sizeof(T)), PL = G;   // lanes per part
  const int NP = 32 / PL;
  T *val = reinterpret_cast<T *>(base);
  uint16_t *col = reinterpret_cast<uint16_t *>(base + (size_t)W * 32 * sizeof(T));
  auto vi = [&](int e, int lane) { return ((e / VE) * 32 + lane) * VE + e % VE; };
  auto ci = [&](int e, int lane) { return ((e / 8) * 32 + lane) * 8 + e % 8; };
  auto pcost = [&](int e, int h) {                                 // wavefronts of part h of column e
    int cnt[16] = {0};
    uint16_t seen[16];
    int ns = 0, m = 0;
    for (int lane = h * PL; lane < (h + 1) * PL; ++lane) {
      const uint16_t sl = col[ci(e, lane)];
      bool dup = false;
      for (int k = 0; k < ns; ++k) dup |= seen[k] == sl;
      if (!dup) {
        seen[ns++] = sl;
        m = std::max(m, ++cnt[sl % G]);
      }
    }
    return m;
  };
  std::vector<int> c((size_t)W * NP);
  int before = 0;
  for (int e = 0; e < W; ++e)
    for (int h = 0; h < NP; ++h) before += (c[e * NP + h] = pcost(e, h));
  for (int pass = 0; pass < 1; ++pass) {                          // further passes gain < 0.01 wavefront
    bool any = false;
    for (int e1 = 0; e1 < W; ++e1)
      for (int h = 0; h < NP; ++h) {
        if (c[e1 * NP + h] <= 1) continue;
        for (int lane = h * PL; lane < (h + 1) * PL && c[e1 * NP + h] > 1; ++lane) {
          // only moving a slot out of a fullest bank group can lower the part's cost
          {
            int cnt[16] = {0};
            uint16_t seen[16];
            int ns = 0;
            for (int l2 = h * PL; l2 < (h + 1) * PL; ++l2) {
              const uint16_t sl = col[ci(e1, l2)];
              bool dup = false;
              for (int k = 0; k < ns; ++k) dup |= seen[k] == sl;
              if (!dup) { seen[ns++] = sl; ++cnt[sl % G]; }
            }
            if (cnt[col[ci(e1, lane)] % G] < c[e1 * NP + h]) continue;
          }
          for (int e2 = 0; e2 < W; ++e2) {
            if (e2 == e1 || (e2 < wo) != (e1 < wo)) continue;        // look-ahead groups stay apart
            uint16_t &s1 = col[ci(e1, lane)], &s2 = col[ci(e2, lane)];
            if (s1 == s2) continue;
            std::swap(s1, s2);
            const int n1 = pcost(e1, h), n2 = pcost(e2, h);
            if (n1 + n2 < c[e1 * NP + h] + c[e2 * NP + h]) {
              std::swap(val[vi(e1, lane)], val[vi(e2, lane)]);
              c[e1 * NP + h] = n1;
              c[e2 * NP + h] = n2;
              any = true;
              break;
            }
            std::swap(s1, s2);
          }
        }
      }
    if (!any) break;
  }
  int after = 0;
  for (int v : c) after += v;
  return {before, after};
}

// Register-prefetched records of the two sweeps (RegPack, k_tri_reg).  Q > 1:
// the split form (plan.hpp), with the chunks of pack_sweep(Q) as its "blocks".
template <typename T>
// Tail form (DESIGN 6b): `sweeps` of any number (each L or U per `up`), Q = 1 only; `lout`
// gives the L sweeps' output positions (per stage row) instead of the U sweep's.
void pack_reg(const std::vector<int64_t> &blk, const std::vector<const TriPack<T> *> &SW, const std::vector<char> &up,
              RegPack<T> &P, int Q = 1, const std::vector<int32_t> *lout = nullptr) {
  P = RegPack<T>();
  P.Q = Q;
  const int NSW = (int)SW.size();
  P.nsweep = NSW;
  if (NSW != 2 && Q > 1) return;                                   // split form: the (L, U) pair only
  if (NSW > 3) return;
  const bool split = Q > 1;
  const TriPack<T> &Lp = *SW[0];
  const TriPack<T> &Up = *SW[NSW - 1];
  static const bool lookahead = getenv("GEMSLR_NO_LOOKAHEAD") == nullptr;   // experiments
  const size_t nblk = blk.size() - 1;
  const size_t nb = nblk * (size_t)Q;                              // pack "blocks" (chunks)
  const int64_t R0 = blk.front(), NR = blk.back() - blk.front();
  P.lslices = (int64_t)Lp.slice_row.size() / 32;
  P.uslices = (int64_t)Up.slice_row.size() / 32;
  for (int k = 0; k < NSW; ++k) P.sw_slices.push_back((int64_t)SW[k]->slice_row.size() / 32);
  for (const TriPack<T> *S : SW)
    for (size_t s = 0; s + 1 < S->slice_off.size(); ++s)
      P.wmax = std::max(P.wmax, (int)((S->slice_off[s + 1] - S->slice_off[s]) / 32));
  P.W = reg_width(std::max(P.wmax, 1));
  if (P.W == 0) return;
  const int W = P.W, W8 = (W + 7) / 8, VE = 16 / (int)sizeof(T);
  P.nrec = 0;
  for (int64_t v : P.sw_slices) P.nrec += v;
  // packed position (stage slice * 32 + lane) of every row in each sweep
  std::vector<std::vector<int32_t>> spos(NSW, std::vector<int32_t>(NR, -1));
  for (int k = 0; k < NSW; ++k)
    for (int64_t s = 0; s < P.sw_slices[k]; ++s)
      for (int lane = 0; lane < 32; ++lane) {
        const int32_t row = SW[k]->slice_row[s * 32 + lane];
        if (row >= 0) spos[k][row - R0] = (int32_t)(s * 32 + lane);
      }
  P.lpos = spos[0];
  const std::vector<int32_t> &upos = spos[NSW - 1];
  // chunk of every stage row (the chunk's rows: pack_sweep's n q / Q split)
  std::vector<int32_t> chunk(NR, 0);
  for (size_t b = 0; b < nblk; ++b) {
    const int64_t n = blk[b + 1] - blk[b];
    for (int q = 0; q < Q; ++q)
      for (int64_t i = n * q / Q; i < n * (q + 1) / Q; ++i) chunk[blk[b] - R0 + i] = (int32_t)(b * Q + q);
  }
  // slice -> (chunk, local level) of each sweep, for the producer side of imports
  std::vector<int32_t> sl_chunk[3], sl_lev[3];
  for (int sweep = 0; sweep < NSW; ++sweep) {
    const TriPack<T> &S = *SW[sweep];
    const int64_t ns = (int64_t)S.slice_row.size() / 32;
    sl_chunk[sweep].assign(ns, 0);
    sl_lev[sweep].assign(ns, 0);
    for (size_t c = 0; c < nb; ++c)
      for (int32_t v = S.blk_lev[c]; v < S.blk_lev[c + 1]; ++v)
        for (int32_t sl = S.lev_slice[v]; sl < S.lev_slice[v + 1]; ++sl) {
          sl_chunk[sweep][sl] = (int32_t)c;
          sl_lev[sweep][sl] = v - S.blk_lev[c];
        }
  }
  // solution window: the smallest power of two covering every (in-chunk)
  // dependency distance (level end - dependency position)
  int64_t need = 1;
  for (size_t b = 0; b < nb; ++b)
    for (int sweep = 0; sweep < NSW; ++sweep) {
      const TriPack<T> &S = *SW[sweep];
      const int32_t lv0 = S.blk_lev[b], lv1 = S.blk_lev[b + 1];
      const int32_t sb0 = S.lev_slice[lv0];
      for (int32_t v = lv0; v < lv1; ++v) {
        const int64_t send = S.lev_slice[v + 1] - sb0;
        for (int64_t g = S.slice_off[S.lev_slice[v]]; g < S.slice_off[S.lev_slice[v + 1]]; ++g) {
          const int32_t dep = S.col[g];
          if (dep < 0 || chunk[dep - R0] != (int32_t)b || spos[sweep][dep - R0] < 0) continue;   // (cross: imports)
          const int32_t q = spos[sweep][dep - R0] - sb0 * 32;
          need = std::max(need, send * 32 - q);
        }
      }
    }
  P.ring = 1024;
  while (P.ring < need && P.ring < REG_RING_BYTES / (int)sizeof(T)) P.ring *= 2;
  // import mode: the tail form, or a one-CTA pack whose dependencies reach further back
  // than the largest ring (a tail-ordered block's full sweeps)
  const bool xmode = NSW == 3 || (!split && need > REG_RING_BYTES / (int)sizeof(T));
  P.xmode = xmode;
  const bool xf = split || xmode;                                  // records carry exp[32]
  P.rec_bytes = reg_record_bytes<T>(W, xf);
  P.data.assign((size_t)P.nrec * P.rec_bytes, 0);
  // tail form: a dependency further back than the ring ("far") or on an earlier sweep
  // ("cross") reads an import slot R + i that its producing lane writes (exp); R is
  // chosen to minimise R + imports (the shared memory of the block's values)
  auto prod_of = [&](int sweep, int32_t dep) {                     // the latest sweep <= `sweep` holding the row
    for (int k = sweep; k >= 0; --k)
      if (spos[k][dep - R0] >= 0) return k;
    return -1;
  };
  auto xkey = [&](int ps, int32_t dep) { return (int64_t)ps * (NR + 1) + (dep - R0); };
  // (producer sweep, dep row) -> widest window of its readers (-1: read by a later sweep,
  // -2: not read); rows belong to one block, so the tables are stage-wide
  std::vector<int64_t> dwin;
  if (xmode) {
    dwin.assign((size_t)NSW * (NR + 1), -2);
    for (size_t b = 0; b < nb; ++b)
      for (int sweep = 0; sweep < NSW; ++sweep) {
        const TriPack<T> &S = *SW[sweep];
        const int32_t lv0 = S.blk_lev[b], lv1 = S.blk_lev[b + 1];
        const int32_t sb0 = S.lev_slice[lv0];
        for (int32_t v = lv0; v < lv1; ++v) {
          const int64_t send = S.lev_slice[v + 1] - sb0;
          for (int64_t g = S.slice_off[S.lev_slice[v]]; g < S.slice_off[S.lev_slice[v + 1]]; ++g) {
            const int32_t dep = S.col[g];
            if (dep < 0) continue;
            if (spos[sweep][dep - R0] < 0) {
              const int ps = prod_of(sweep - 1, dep);
              if (ps < 0) return;                                  // read but never computed
              dwin[xkey(ps, dep)] = -1;
              continue;
            }
            int64_t &w = dwin[xkey(sweep, dep)];
            if (w == -2) w = 0;
            if (w >= 0) w = std::max<int64_t>(w, send * 32 - (spos[sweep][dep - R0] - sb0 * 32));
          }
        }
      }
    int64_t maxsl = 0;                                             // level table entries of the largest block
    for (size_t b = 0; b < nb; ++b) {
      int64_t t = 0;
      for (const TriPack<T> *S : SW) t += S->lev_slice[S->blk_lev[b + 1]] - S->lev_slice[S->blk_lev[b]];
      maxsl = std::max(maxsl, t);
    }
    int best = -1;
    int64_t bestc = 0;
    for (int r = 1024; r <= REG_RING_BYTES / (int)sizeof(T); r *= 2) {
      int64_t imp = 0;
      for (size_t b = 0; b < nb; ++b) {
        int64_t c = 0;
        for (int k = 0; k < NSW; ++k)
          for (int64_t i = blk[b] - R0; i < blk[b + 1] - R0; ++i) {
            const int64_t w = dwin[xkey(k, (int32_t)(i + R0))];
            c += (w == -1 || w > r) ? 1 : 0;
          }
        imp = std::max(imp, c);
      }
      const int64_t bytes = (r + imp) * (int64_t)sizeof(T) + 16 + (int64_t)al16_h((size_t)maxsl * 2);
      if (r + imp > 65535 || bytes > 232448 - 1024 - 2048) continue;
      if (best < 0 || r + imp <= bestc) { best = r; bestc = r + imp; }
    }
    if (best < 0) return;
    P.ring = best;
  }
  const int R = P.ring;
  // look-ahead (plan.hpp REG_LA): every row's entries on the previous level of its chunk
  // (in-chunk dependencies only; imports are always ready before) must fit REG_LA columns
  {
    int maxnew = 0;
    for (size_t b = 0; b < nb; ++b)
      for (int sweep = 0; sweep < NSW; ++sweep) {
        const TriPack<T> &S = *SW[sweep];
        for (int32_t v = S.blk_lev[b]; v < S.blk_lev[b + 1]; ++v)
          for (int32_t sl = S.lev_slice[v]; sl < S.lev_slice[v + 1]; ++sl) {
            const int w = (int)((S.slice_off[sl + 1] - S.slice_off[sl]) / 32);
            for (int lane = 0; lane < 32; ++lane) {
              int c = 0;
              for (int e = 0; e < w; ++e) {
                const int32_t dep = S.col[S.slice_off[sl] + 32 * e + lane];
                if (dep < 0 || chunk[dep - R0] != (int32_t)b || spos[sweep][dep - R0] < 0) continue;
                const int32_t pd = spos[sweep][dep - R0];
                if (sl_lev[sweep][pd / 32] >= (v - S.blk_lev[b]) - 1) c++;
              }
              maxnew = std::max(maxnew, c);
            }
          }
      }
    // Measured (tools/split_cmp.py, DOWN / UP per apply): the look-ahead shortens the
    // per-level chain where levels carry 1-2 slices (C5 level 1 51.7 -> 47.5 us, C4 level
    // 1 76 -> 70, level 2 23 -> 21) but costs where several slices per level contend for
    // the shared-memory pipe (the two column groups constrain the bank spread of the
    // gathers: C3 level 0 180 -> 199 us, C4 level 0 269 -> 313; C5's split level 0
    // 227 -> 223): so only stages with fewer than 2 slices per level on average.
    int64_t sl = 0, lv = 0;
    for (size_t b = 0; b < nb; ++b) {
      for (const TriPack<T> *S : SW) {
        sl += S->lev_slice[S->blk_lev[b + 1]] - S->lev_slice[S->blk_lev[b]];
        lv += S->blk_lev[b + 1] - S->blk_lev[b];
      }
    }
    const double K = lv > 0 ? (double)sl / (double)lv : 1.0;
    P.la = (lookahead && maxnew <= REG_LA && W > REG_LA && K < 2.0) ? REG_LA : 0;
  }
  // split: imports of every chunk and sweep (dependency rows in another chunk),
  // numbered in the order the consumer's records first need them
  std::vector<std::vector<std::pair<int32_t, int32_t>>> imp[2];   // per chunk: (stage row, producer slice)
  if (split) {
    for (int sweep = 0; sweep < 2; ++sweep) {
      const TriPack<T> &S = sweep ? Up : Lp;
      imp[sweep].assign(nb, {});
      std::vector<int32_t> seen(NR, -1);
      for (size_t b = 0; b < nb; ++b)
        for (int64_t g = S.slice_off[S.lev_slice[S.blk_lev[b]]]; g < S.slice_off[S.lev_slice[S.blk_lev[b + 1]]]; ++g) {
          const int32_t dep = S.col[g];
          if (dep < 0) continue;
          const int32_t pc = chunk[dep - R0];
          if (pc == (int32_t)b) continue;
          // one-directional chains only: L from chunk q - 1, U from q + 1 of the same block
          if (pc / Q != (int32_t)b / Q || pc != (int32_t)b + (sweep ? 1 : -1)) return;
          if (seen[dep - R0] == (int32_t)b) continue;
          seen[dep - R0] = (int32_t)b;
          const int32_t pslice = (sweep ? upos[dep - R0] : P.lpos[dep - R0]) / 32;
          imp[sweep][b].push_back({dep - (int32_t)R0, pslice});
        }
    }
    for (size_t b = 0; b < nb; ++b) {
      P.imp_L = std::max(P.imp_L, (int)imp[0][b].size());
      P.imp_U = std::max(P.imp_U, (int)imp[1][b].size());
    }
    if ((int64_t)R + P.imp_L + P.imp_U > 65535) return;
  }
  // tail form: the far and cross rows of every block get import slots, numbered in the
  // order the consumers' records first need them; the producer is the latest sweep up to
  // the consumer's holding the row
  std::vector<int32_t> xmap;                                       // (producer sweep, row) -> index in its block
  std::vector<std::vector<std::pair<int32_t, int32_t>>> xprod;     // per block: (producer sweep, position)
  auto is_imp = [&](size_t, int ps, int32_t dep) {
    const int64_t w = dwin[xkey(ps, dep)];
    return w == -1 || w > R;
  };
  if (xmode) {
    xmap.assign((size_t)NSW * (NR + 1), -1);
    xprod.resize(nb);
    for (size_t b = 0; b < nb; ++b)
      for (int sweep = 0; sweep < NSW; ++sweep) {
        const TriPack<T> &S = *SW[sweep];
        for (int64_t g = S.slice_off[S.lev_slice[S.blk_lev[b]]]; g < S.slice_off[S.lev_slice[S.blk_lev[b + 1]]]; ++g) {
          const int32_t dep = S.col[g];
          if (dep < 0) continue;
          const int ps = sweep > 0 && spos[sweep][dep - R0] < 0 ? prod_of(sweep - 1, dep) : sweep;
          if (ps < 0) return;                                      // read but never computed
          if (!is_imp(b, ps, dep)) continue;
          if (xmap[xkey(ps, dep)] >= 0) continue;
          xmap[xkey(ps, dep)] = (int32_t)xprod[b].size();
          xprod[b].push_back({ps, spos[ps][dep - R0]});
        }
      }
    for (size_t b = 0; b < nb; ++b) P.imp_L = std::max(P.imp_L, (int)xprod[b].size());
    if ((int64_t)R + P.imp_L > 65535) return;
  }
  // per chunk and sweep: stage row -> import index (only rows imported by that chunk)
  std::vector<std::unordered_map<int32_t, int32_t>> impmap[2];
  if (split)
    for (int sweep = 0; sweep < 2; ++sweep) {
      impmap[sweep].resize(nb);
      for (size_t b = 0; b < nb; ++b)
        for (size_t i = 0; i < imp[sweep][b].size(); ++i) impmap[sweep][b][imp[sweep][b][i].first] = (int32_t)i;
    }
  std::vector<int64_t> rec_of[3];                                  // stage slice -> record
  for (int k = 0; k < NSW; ++k) rec_of[k].assign(P.sw_slices[k], -1);
  // Records are numbered and their bookkeeping done in order; their contents are then
  // filled in parallel (independent records).
  struct Task { int64_t rec; int32_t b; int sweep; int32_t v, s, lv0, sb0, send; };
  std::vector<Task> tasks;
  tasks.reserve((size_t)P.nrec);
  auto fill = [&](const Task &tk, int64_t &nearc, int64_t &farc) {
    const int64_t rec = tk.rec;
    const size_t b = (size_t)tk.b;
    const int sweep = tk.sweep;
    const int32_t v = tk.v, s = tk.s, lv0 = tk.lv0, sb0 = tk.sb0, send = tk.send;
    const TriPack<T> &S = *SW[sweep];
    const bool upper = up[sweep] != 0;
    const int w = (int)((S.slice_off[s + 1] - S.slice_off[s]) / 32);
    uint8_t *base = P.data.data() + (size_t)rec * P.rec_bytes;
    T *val = reinterpret_cast<T *>(base);
    uint16_t *col = reinterpret_cast<uint16_t *>(base + (size_t)W * 32 * sizeof(T));
    int32_t *out = reinterpret_cast<int32_t *>(col + (size_t)W8 * 32 * 8);
    T *rdiag = reinterpret_cast<T *>(out + 32);
    if (xf) {
      int32_t *exp = reinterpret_cast<int32_t *>(rdiag + 32);
      for (int lane = 0; lane < 32; ++lane) exp[lane] = -1;
    }
    // entries of every lane with their ring slots, split for the look-ahead:
    // "new" = a dependency in the immediately preceding level of this chunk
    // (needs that level's barrier), "old" = older levels and imports (ready after
    // the barrier before it, so k_tri_reg sums them while the previous level runs)
    struct Ent { T v; uint16_t slot; bool nw; };
    std::vector<Ent> ent[32];
    for (int lane = 0; lane < 32; ++lane) {
      const int32_t row = S.slice_row[(int64_t)s * 32 + lane];
      out[lane] = row < 0 ? -1 : (upper ? row : lout ? (*lout)[row - R0] : upos[row - R0]);
      rdiag[lane] = upper ? T(1) / S.diag[(int64_t)s * 32 + lane] : T(1);
      for (int e = 0; e < w; ++e) {
        const int64_t g = S.slice_off[s] + 32 * e + lane;
        const int32_t dep = S.col[g];
        if (dep < 0) continue;
        if (split && chunk[dep - R0] != (int32_t)b) {         // an import (DSMEM from the neighbour chunk)
          const int32_t ii = impmap[sweep][b].at(dep - (int32_t)R0);
          const int32_t pslice = imp[sweep][b][ii].second;
          (void)pslice;
          ent[lane].push_back(Ent{S.val[g], (uint16_t)(R + (upper ? P.imp_L : 0) + ii), false});
          nearc++;
          continue;
        }
        if (NSW == 3 && spos[sweep][dep - R0] < 0) {           // cross: from an earlier sweep
          ent[lane].push_back(Ent{S.val[g], (uint16_t)(R + xmap[xkey(prod_of(sweep - 1, dep), dep)]), false});
          nearc++;
          continue;
        }
        const int32_t pd = spos[sweep][dep - R0];
        const int32_t q = pd - sb0 * 32;                  // block-relative position
        const bool isnew = sl_lev[sweep][pd / 32] >= (v - lv0) - 1;
        if (xmode && is_imp(b, sweep, dep)) {               // far: an import slot
          ent[lane].push_back(Ent{S.val[g], (uint16_t)(R + xmap[xkey(sweep, dep)]), isnew});
          nearc++;
          continue;
        }
        if ((int64_t)send * 32 - 1 - q < R) { ent[lane].push_back(Ent{S.val[g], (uint16_t)(q & (R - 1)), isnew}); nearc++; }
        else { farc++; }
      }
    }
    // look-ahead groups: columns [0, wo) old, [wo, W) new (wo = W - la); a lane's
    // old entries beyond wo fill its unused new columns (old + new <= W)
    const int wo = W - P.la;
    std::vector<Ent> grp[2][32];
    for (int lane = 0; lane < 32; ++lane) {
      for (const Ent &en : ent[lane])
        if (P.la == 0 || (!en.nw && (int)grp[0][lane].size() < wo)) grp[0][lane].push_back(en);
        else grp[1][lane].push_back(en);
    }
    // Column e of the slice is one shared-memory gather of 32 lanes (8 or 16
    // bytes each); order each lane's entries (any order gives the same sum up
    // to rounding) so that every column spreads its distinct slots over the
    // bank groups: greedily give each lane the entry whose group is least
    // used in the column so far.
    // Counted per part of the warp the LDS serves in one pass (16 lanes for
    // 8-byte slots, 8 for 16-byte; see refine_record).
    const int G = (int)(128 / sizeof(T));                 // bank groups of one 128-byte wavefront
    for (int e = 0; e < W; ++e) {
      std::vector<int> cnt(G, 0);
      std::vector<uint16_t> seen;
      for (int lane = 0; lane < 32; ++lane) {
        if (lane % G == 0) {                              // a new part of the warp
          std::fill(cnt.begin(), cnt.end(), 0);
          seen.clear();
        }
        uint16_t slot = (uint16_t)(R - 1);
        T v = T(0);
        auto &L = grp[P.la == 0 || e < wo ? 0 : 1][lane];
        if (!L.empty()) {
          size_t best = 0;
          int bc = 1 << 30;
          for (size_t k = 0; k < L.size(); ++k) {
            const bool dup = std::find(seen.begin(), seen.end(), L[k].slot) != seen.end();
            const int c = dup ? -1 : cnt[L[k].slot % G];          // a repeated slot is a broadcast
            if (c < bc) { bc = c; best = k; }
          }
          slot = L[best].slot;
          v = L[best].v;
          L.erase(L.begin() + (long)best);
        }
        if (std::find(seen.begin(), seen.end(), slot) == seen.end()) {
          seen.push_back(slot);
          cnt[slot % G]++;
        }
        val[((e / VE) * 32 + lane) * VE + e % VE] = v;
        col[((e / 8) * 32 + lane) * 8 + e % 8] = slot;
      }
    }
  };
  int64_t rec = 0;
  for (size_t b = 0; b < nb; ++b) {
    int32_t info[REG_BINFO_INTS] = {0};
    const size_t bk = b / (size_t)Q;                               // original block
    const int64_t nbk = blk[bk + 1] - blk[bk];
    const int qq = (int)(b % (size_t)Q);
    info[8] = (int32_t)(blk[bk] + nbk * qq / Q);                   // this chunk's rows
    info[9] = (int32_t)(blk[bk] + nbk * (qq + 1) / Q);
    for (int sweep = 0; sweep < NSW; ++sweep) {
      const TriPack<T> &S = *SW[sweep];
      const bool upper = up[sweep] != 0;
      const int32_t lv0 = S.blk_lev[b], lv1 = S.blk_lev[b + 1];
      const int32_t sb0 = S.lev_slice[lv0];
      info[3 * sweep + 0] = (int32_t)rec;
      info[3 * sweep + 1] = S.lev_slice[lv1] - sb0;
      info[3 * sweep + 2] = lv1 - lv0;
      if (NSW == 2) {
        info[6 + sweep] = (int32_t)P.lev_off.size();
        info[10 + sweep] = sb0;
      } else {
        info[9 + sweep] = sb0;                                     // tail layout (plan.hpp)
      }
      P.max_levels = std::max(P.max_levels, lv1 - lv0);
      int need_pref = -1;                                          // split: producer level needed so far
      for (int32_t v = lv0; v < lv1; ++v) {
        P.lev_off.push_back((int32_t)rec);
        const int32_t send = S.lev_slice[v + 1] - sb0;     // level end (block-relative slice)
        for (int32_t s = S.lev_slice[v]; s < S.lev_slice[v + 1]; ++s, ++rec) {
          rec_of[sweep][s] = rec;
          if (v - lv0 > 65535) return;
          P.slev.push_back((uint16_t)(v - lv0));
          if (split) {                                             // producer level of the imports read so far
            const int w = (int)((S.slice_off[s + 1] - S.slice_off[s]) / 32);
            for (int64_t g = S.slice_off[s]; g < S.slice_off[s] + 32 * w; ++g) {
              const int32_t dep = S.col[g];
              if (dep < 0 || chunk[dep - R0] == (int32_t)b) continue;
              auto it = impmap[sweep][b].find(dep - (int32_t)R0);
              if (it == impmap[sweep][b].end()) return;
              need_pref = std::max(need_pref, sl_lev[sweep][imp[sweep][b][it->second].second]);
            }
            P.sneed.push_back((uint16_t)(need_pref + 1));
          }
          tasks.push_back(Task{rec, (int32_t)b, sweep, v, s, lv0, sb0, send});
        }
      }
      P.lev_off.push_back((int32_t)rec);
    }
    P.binfo.insert(P.binfo.end(), info, info + REG_BINFO_INTS);
    P.max_block_slices = std::max(P.max_block_slices, info[1] + info[4] + (NSW == 3 ? info[7] : 0));
  }
  {
    int64_t nearc = 0, farc = 0;
#pragma omp parallel for schedule(dynamic, 64) reduction(+ : nearc, farc)
    for (int64_t t = 0; t < (int64_t)tasks.size(); ++t) fill(tasks[(size_t)t], nearc, farc);
    P.near += nearc;
    P.far += farc;
  }
  if (split) {
    // exports: the producer lane of every import, and per producer chunk and sweep
    // the number of values exported at each local level (the bytes the consumer's
    // barrier of that level awaits); binfo[12..15] of the CONSUMER point at its
    // producers' tables
    std::vector<int32_t> xoff[2];
    for (int sweep = 0; sweep < 2; ++sweep) {
      const TriPack<T> &S = sweep ? Up : Lp;
      xoff[sweep].assign(nb, 0);
      std::vector<std::vector<uint16_t>> tab(nb);
      for (size_t c = 0; c < nb; ++c) tab[c].assign(S.blk_lev[c + 1] - S.blk_lev[c], 0);
      for (size_t b = 0; b < nb; ++b)
        for (size_t i = 0; i < imp[sweep][b].size(); ++i) {
          const int32_t row = imp[sweep][b][i].first, ps = imp[sweep][b][i].second;
          const int32_t pd = sweep ? upos[row] : P.lpos[row];
          const int64_t r = rec_of[sweep][ps];
          uint8_t *base = P.data.data() + (size_t)r * P.rec_bytes;
          int32_t *exp = reinterpret_cast<int32_t *>(base + (size_t)W * 32 * sizeof(T) + (size_t)W8 * 512 + 32 * 4 +
                                                     32 * sizeof(T));
          if (exp[pd % 32] >= 0) return;                           // exported to two chunks: not supported
          exp[pd % 32] = (int32_t)i;
          P.exports++;
          uint16_t &t = tab[sl_chunk[sweep][ps]][sl_lev[sweep][ps]];   // values the consumer's barrier awaits
          if (t == 65535) return;
          t++;
        }
      for (size_t c = 0; c < nb; ++c) {
        xoff[sweep][c] = (int32_t)P.xexp.size();
        P.xexp.insert(P.xexp.end(), tab[c].begin(), tab[c].end());
        (sweep ? P.plev_U : P.plev_L) = std::max(sweep ? P.plev_U : P.plev_L, (int)tab[c].size());
      }
    }
    for (size_t b = 0; b < nb; ++b) {
      int32_t *info = &P.binfo[b * REG_BINFO_INTS];
      const int qq = (int)(b % (size_t)Q);
      if (qq > 0) { info[12] = xoff[0][b - 1]; info[13] = Lp.blk_lev[b] - Lp.blk_lev[b - 1]; }
      if (qq + 1 < Q) { info[14] = xoff[1][b + 1]; info[15] = Up.blk_lev[b + 2] - Up.blk_lev[b + 1]; }
    }
  }
  if (xmode) {                                                    // producer lanes of the imports
    for (size_t b = 0; b < nb; ++b)
      for (size_t i = 0; i < xprod[b].size(); ++i) {
        const int ps = xprod[b][i].first, pd = xprod[b][i].second;
        const int64_t r = rec_of[ps][pd / 32];
        uint8_t *base = P.data.data() + (size_t)r * P.rec_bytes;
        int32_t *exp = reinterpret_cast<int32_t *>(base + (size_t)W * 32 * sizeof(T) + (size_t)W8 * 512 + 32 * 4 +
                                                   32 * sizeof(T));
        exp[pd % 32] = (int32_t)i;
        P.exports++;
      }
  }
  {
    long long cb = 0, ca = 0;
#pragma omp parallel for schedule(dynamic, 256) reduction(+ : cb, ca)
    for (int64_t r = 0; r < P.nrec; ++r) {
      const auto ba = refine_record<T>(P.data.data() + (size_t)r * P.rec_bytes, W, W - P.la);
      cb += ba.first;
      ca += ba.second;
    }
    if (getenv("GEMSLR_DEBUG_BANKS"))
      fprintf(stderr, "gathers: %.3f -> %.3f wavefronts per LDS (%lld records, W %d)\n",
              (double)cb / std::max<int64_t>(P.nrec * W, 1), (double)ca / std::max<int64_t>(P.nrec * W, 1),
              (long long)P.nrec, W);
  }
  P.ok = P.far == 0 && R <= 65536 && P.nrec < INT32_MAX;
}

}  // namespace

// Tail form of the sweeps (plan.hpp TailPack, DESIGN 6b), one CTA per block.
template <typename T>
void pack_tail(const std::vector<int64_t> &blk, const std::vector<Factor<T>> &fac, const std::vector<int64_t> &tails,
               TailPack<T> &TP) {
  TP = TailPack<T>();
  const size_t nb = fac.size();
  if (tails.size() != nb || nb == 0) return;
  std::vector<int64_t> ts(nb);
  for (size_t b = 0; b < nb; ++b) {
    ts[b] = std::min(std::max(tails[b], blk[b]), blk[b + 1]) - blk[b];
    TP.tail_rows += blk[b + 1] - blk[b] - ts[b];
  }
  TP.ts = tails;
  pack_sweep(blk, fac, false, TP.Lhh, 1, 1, &ts);                 // head rows of L
  pack_sweep(blk, fac, false, TP.Lth, 1, 2, &ts, true);           // tail rows of L (head columns: cross)
  pack_sweep(blk, fac, true, TP.Utt, 1, 2, &ts);                  // tail rows of U
  pack_sweep(blk, fac, true, TP.Uht, 1, 1, &ts, true);            // head rows of U (tail columns: cross)
  pack_sweep(blk, fac, false, TP.Ltt, 1, 2, &ts);                 // tail rows of L, head columns dropped
  const int64_t R0 = blk.front(), NR = blk.back() - blk.front();
  auto posof = [&](const TriPack<T> &S, std::vector<int32_t> &pos, int32_t off) {
    for (size_t q = 0; q < S.slice_row.size(); ++q)
      if (S.slice_row[q] >= 0) pos[S.slice_row[q] - R0] = off + (int32_t)q;
  };
  const int32_t nUtt = (int32_t)TP.Utt.slice_row.size(), nLhh = (int32_t)TP.Lhh.slice_row.size();
  TP.nUtt = nUtt;
  TP.nLhh = nLhh;
  TP.ucat.assign(NR, -1);
  posof(TP.Utt, TP.ucat, 0);
  posof(TP.Uht, TP.ucat, nUtt);
  TP.lcat.assign(NR, -1);
  posof(TP.Lhh, TP.lcat, 0);
  posof(TP.Lth, TP.lcat, nLhh);
  TP.uttpos.assign(NR, -1);
  posof(TP.Utt, TP.uttpos, 0);
  TP.lttpos.assign(NR, -1);
  posof(TP.Ltt, TP.lttpos, 0);
  TP.lrow = TP.Lhh.slice_row;
  TP.lrow.insert(TP.lrow.end(), TP.Lth.slice_row.begin(), TP.Lth.slice_row.end());
  const auto c0 = std::chrono::steady_clock::now();
  pack_reg(blk, {&TP.Lhh, &TP.Lth, &TP.Utt}, {0, 0, 1}, TP.D, 1, &TP.ucat);
  const auto c1 = std::chrono::steady_clock::now();
  pack_reg(blk, {&TP.Ltt, &TP.Utt, &TP.Uht}, {0, 1, 1}, TP.U, 1, &TP.ucat);
  if (getenv("GEMSLR_DEBUG_TAIL"))
    fprintf(stderr, "pack_reg D %.2f s U %.2f s\n", std::chrono::duration<double>(c1 - c0).count(),
            std::chrono::duration<double>(std::chrono::steady_clock::now() - c1).count());
  TP.ok = TP.D.ok && TP.U.ok;
  if (getenv("GEMSLR_DEBUG_TAIL"))
    for (const RegPack<T> *R : {&TP.D, &TP.U})
      fprintf(stderr, "tail pack: ok %d ring %d imports %d W %d la %d far %lld records %lld max_block_slices %d\n",
              (int)R->ok, R->ring, R->imp_L, R->W, R->la, (long long)R->far, (long long)R->nrec, R->max_block_slices);
}

// Q > 1: the split form (every block's sweeps over a Q-CTA cluster); when it
// cannot be built (a dependency two chunks away, too many imports) the stage
// falls back to Q / 2, down to the one-CTA form.  The split form has no TMA /
// level-kernel variant (their blocks must be independent).  tails: the tail form
// as well (one CTA per block).
template <typename T>
void pack_stage(const std::vector<int64_t> &blk, const std::vector<Factor<T>> &fac, Stage<T> &S, int Q,
                const std::vector<int64_t> *tails) {
  S.blk = blk;
  S.tail = TailPack<T>();
  const auto t0 = std::chrono::steady_clock::now();
  if (tails) pack_tail(blk, fac, *tails, S.tail);
  if (getenv("GEMSLR_DEBUG_TAIL"))
    fprintf(stderr, "pack_tail %.2f s\n", std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count());
  // a tail-ordered block's tail rows read every chunk: no split form
  if (S.tail.ok) Q = 1;
  for (; Q > 1; Q /= 2) {
    pack_sweep(blk, fac, false, S.Lp, Q);
    pack_sweep(blk, fac, true, S.Up, Q);
    pack_reg(blk, {&S.Lp, &S.Up}, {0, 1}, S.reg, Q);
    if (S.reg.ok) {
      S.pipe = PipePack<T>();
      return;
    }
  }
  pack_sweep(blk, fac, false, S.Lp);
  pack_sweep(blk, fac, true, S.Up);
  pack_pipe(blk, S.Lp, S.Up, S.pipe);
  pack_reg(blk, {&S.Lp, &S.Up}, {0, 1}, S.reg);
  if (getenv("GEMSLR_DEBUG_TAIL"))
    fprintf(stderr, "full pack: ok %d ring %d imports %d xmode %d W %d\n", (int)S.reg.ok, S.reg.ring, S.reg.imp_L,
            (int)S.reg.xmode, S.reg.W);
}

template void pack_stage<double>(const std::vector<int64_t> &, const std::vector<Factor<double>> &, Stage<double> &, int,
                                 const std::vector<int64_t> *);
template void pack_stage<zc>(const std::vector<int64_t> &, const std::vector<Factor<zc>> &, Stage<zc> &, int,
                             const std::vector<int64_t> *);

}  // namespace gemslr
