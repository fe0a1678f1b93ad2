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
#include <unordered_map>

#include "plan.hpp"

namespace gemslr {

namespace {

// Q > 1 (split form, plan.hpp RegPack): block b is packed as Q chunks of
// contiguous rows, each with the levels of the whole block's DAG in which it has
// rows; "block" b Q + q of the pack is chunk q of block b.
template <typename T>
void pack_sweep(const std::vector<int64_t> &blk, const std::vector<Factor<T>> &fac, bool upper, TriPack<T> &P,
                int Q = 1) {
  P = TriPack<T>();
  P.blk_lev.push_back(0);
  P.lev_slice.push_back(0);
  P.slice_off.push_back(0);
  const size_t nb = fac.size();
  for (size_t b = 0; b < nb; ++b) {
    const Csr<T> &M = upper ? fac[b].U : fac[b].L;
    const int64_t n = M.n;
    const int64_t row0 = blk[b];
    std::vector<int32_t> lev(n, 0);
    int32_t nlev = 0;
    if (!upper) {
      for (int64_t i = 0; i < n; ++i) {
        int32_t v = 0;
        for (int64_t p = M.ptr[i]; p < M.ptr[i + 1]; ++p) v = std::max(v, lev[M.col[p]] + 1);
        lev[i] = v;
        nlev = std::max(nlev, v + 1);
      }
    } else {
      for (int64_t i = n - 1; i >= 0; --i) {
        int32_t v = 0;
        for (int64_t p = M.ptr[i] + 1; p < M.ptr[i + 1]; ++p) v = std::max(v, lev[M.col[p]] + 1);
        lev[i] = v;
        nlev = std::max(nlev, v + 1);
      }
    }
    if (n == 0) nlev = 0;
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
    for (int64_t i = c0; i < c1; ++i) cnt[lev[i] + 1]++;
    for (int32_t v = 0; v < nlev; ++v) cnt[v + 1] += cnt[v];
    std::vector<int64_t> rows(c1 - c0);
    {
      std::vector<int64_t> pos(cnt.begin(), cnt.end() - 1);
      for (int64_t i = c0; i < c1; ++i) rows[pos[lev[i]]++] = i;
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
          int64_t len = M.ptr[i + 1] - M.ptr[i] - (upper ? 1 : 0);
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
          for (int64_t p = pb, e = 0; p < M.ptr[i + 1]; ++p, ++e) {
            P.col[off + 32 * e + lane] = (int32_t)(row0 + M.col[p]);
            P.val[off + 32 * e + lane] = M.val[p];
            P.nnz_real++;
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
void pack_reg(const std::vector<int64_t> &blk, const TriPack<T> &Lp, const TriPack<T> &Up, RegPack<T> &P, int Q = 1) {
  P = RegPack<T>();
  P.Q = Q;
  const bool split = Q > 1;
  static const bool lookahead = getenv("GEMSLR_NO_LOOKAHEAD") == nullptr;   // experiments
  const size_t nblk = blk.size() - 1;
  const size_t nb = nblk * (size_t)Q;                              // pack "blocks" (chunks)
  const int64_t R0 = blk.front(), NR = blk.back() - blk.front();
  P.lslices = (int64_t)Lp.slice_row.size() / 32;
  P.uslices = (int64_t)Up.slice_row.size() / 32;
  for (const TriPack<T> *S : {&Lp, &Up})
    for (size_t s = 0; s + 1 < S->slice_off.size(); ++s)
      P.wmax = std::max(P.wmax, (int)((S->slice_off[s + 1] - S->slice_off[s]) / 32));
  P.W = reg_width(std::max(P.wmax, 1));
  if (P.W == 0) return;
  const int W = P.W, W8 = (W + 7) / 8, VE = 16 / (int)sizeof(T);
  P.rec_bytes = reg_record_bytes<T>(W, split);
  P.nrec = P.lslices + P.uslices;
  P.data.assign((size_t)P.nrec * P.rec_bytes, 0);
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
  // chunk of every stage row (the chunk's rows: pack_sweep's n q / Q split)
  std::vector<int32_t> chunk(NR, 0);
  for (size_t b = 0; b < nblk; ++b) {
    const int64_t n = blk[b + 1] - blk[b];
    for (int q = 0; q < Q; ++q)
      for (int64_t i = n * q / Q; i < n * (q + 1) / Q; ++i) chunk[blk[b] - R0 + i] = (int32_t)(b * Q + q);
  }
  // slice -> (chunk, local level) of each sweep, for the producer side of imports
  std::vector<int32_t> sl_chunk[2], sl_lev[2];
  for (int sweep = 0; sweep < 2; ++sweep) {
    const TriPack<T> &S = sweep ? Up : Lp;
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
    for (int sweep = 0; sweep < 2; ++sweep) {
      const TriPack<T> &S = sweep ? Up : Lp;
      const int32_t lv0 = S.blk_lev[b], lv1 = S.blk_lev[b + 1];
      const int32_t sb0 = S.lev_slice[lv0];
      for (int32_t v = lv0; v < lv1; ++v) {
        const int64_t send = S.lev_slice[v + 1] - sb0;
        for (int64_t g = S.slice_off[S.lev_slice[v]]; g < S.slice_off[S.lev_slice[v + 1]]; ++g) {
          const int32_t dep = S.col[g];
          if (dep < 0 || chunk[dep - R0] != (int32_t)b) continue;
          const int32_t q = (sweep ? upos[dep - R0] : P.lpos[dep - R0]) - sb0 * 32;
          need = std::max(need, send * 32 - q);
        }
      }
    }
  P.ring = 1024;
  while (P.ring < need && P.ring < REG_RING_BYTES / (int)sizeof(T)) P.ring *= 2;
  const int R = P.ring;
  // look-ahead (plan.hpp REG_LA): every row's entries on the previous level of its chunk
  // (in-chunk dependencies only; imports are always ready before) must fit REG_LA columns
  {
    int maxnew = 0;
    for (size_t b = 0; b < nb; ++b)
      for (int sweep = 0; sweep < 2; ++sweep) {
        const TriPack<T> &S = sweep ? Up : Lp;
        for (int32_t v = S.blk_lev[b]; v < S.blk_lev[b + 1]; ++v)
          for (int32_t sl = S.lev_slice[v]; sl < S.lev_slice[v + 1]; ++sl) {
            const int w = (int)((S.slice_off[sl + 1] - S.slice_off[sl]) / 32);
            for (int lane = 0; lane < 32; ++lane) {
              int c = 0;
              for (int e = 0; e < w; ++e) {
                const int32_t dep = S.col[S.slice_off[sl] + 32 * e + lane];
                if (dep < 0 || chunk[dep - R0] != (int32_t)b) continue;
                const int32_t pd = sweep ? upos[dep - R0] : P.lpos[dep - R0];
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
      sl += (Lp.lev_slice[Lp.blk_lev[b + 1]] - Lp.lev_slice[Lp.blk_lev[b]]) +
            (Up.lev_slice[Up.blk_lev[b + 1]] - Up.lev_slice[Up.blk_lev[b]]);
      lv += (Lp.blk_lev[b + 1] - Lp.blk_lev[b]) + (Up.blk_lev[b + 1] - Up.blk_lev[b]);
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
  // per chunk and sweep: stage row -> import index (only rows imported by that chunk)
  std::vector<std::unordered_map<int32_t, int32_t>> impmap[2];
  if (split)
    for (int sweep = 0; sweep < 2; ++sweep) {
      impmap[sweep].resize(nb);
      for (size_t b = 0; b < nb; ++b)
        for (size_t i = 0; i < imp[sweep][b].size(); ++i) impmap[sweep][b][imp[sweep][b][i].first] = (int32_t)i;
    }
  std::vector<int64_t> rec_of[2];                                  // stage slice -> record
  rec_of[0].assign(P.lslices, -1);
  rec_of[1].assign(P.uslices, -1);
  int64_t rec = 0;
  for (size_t b = 0; b < nb; ++b) {
    int32_t info[REG_BINFO_INTS] = {0};
    const size_t bk = b / (size_t)Q;                               // original block
    const int64_t nbk = blk[bk + 1] - blk[bk];
    const int qq = (int)(b % (size_t)Q);
    info[8] = (int32_t)(blk[bk] + nbk * qq / Q);                   // this chunk's rows
    info[9] = (int32_t)(blk[bk] + nbk * (qq + 1) / Q);
    for (int sweep = 0; sweep < 2; ++sweep) {
      const TriPack<T> &S = sweep ? Up : Lp;
      const bool upper = sweep == 1;
      const int32_t lv0 = S.blk_lev[b], lv1 = S.blk_lev[b + 1];
      const int32_t sb0 = S.lev_slice[lv0];
      info[3 * sweep + 0] = (int32_t)rec;
      info[3 * sweep + 1] = S.lev_slice[lv1] - sb0;
      info[3 * sweep + 2] = lv1 - lv0;
      info[6 + sweep] = (int32_t)P.lev_off.size();
      info[10 + sweep] = sb0;
      P.max_levels = std::max(P.max_levels, lv1 - lv0);
      int need_pref = -1;                                          // split: producer level needed so far
      for (int32_t v = lv0; v < lv1; ++v) {
        P.lev_off.push_back((int32_t)rec);
        const int32_t send = S.lev_slice[v + 1] - sb0;     // level end (block-relative slice)
        for (int32_t s = S.lev_slice[v]; s < S.lev_slice[v + 1]; ++s, ++rec) {
          const int w = (int)((S.slice_off[s + 1] - S.slice_off[s]) / 32);
          uint8_t *base = P.data.data() + (size_t)rec * P.rec_bytes;
          T *val = reinterpret_cast<T *>(base);
          uint16_t *col = reinterpret_cast<uint16_t *>(base + (size_t)W * 32 * sizeof(T));
          int32_t *out = reinterpret_cast<int32_t *>(col + (size_t)W8 * 32 * 8);
          T *rdiag = reinterpret_cast<T *>(out + 32);
          if (split) {
            int32_t *exp = reinterpret_cast<int32_t *>(rdiag + 32);
            for (int lane = 0; lane < 32; ++lane) exp[lane] = -1;
          }
          rec_of[sweep][s] = rec;
          if (v - lv0 > 65535) return;
          P.slev.push_back((uint16_t)(v - lv0));
          // entries of every lane with their ring slots, split for the look-ahead:
          // "new" = a dependency in the immediately preceding level of this chunk
          // (needs that level's barrier), "old" = older levels and imports (ready after
          // the barrier before it, so k_tri_reg sums them while the previous level runs)
          struct Ent { T v; uint16_t slot; bool nw; };
          std::vector<Ent> ent[32];
          for (int lane = 0; lane < 32; ++lane) {
            const int32_t row = S.slice_row[(int64_t)s * 32 + lane];
            out[lane] = row < 0 ? -1 : (upper ? row : upos[row - R0]);
            rdiag[lane] = upper ? T(1) / S.diag[(int64_t)s * 32 + lane] : T(1);
            for (int e = 0; e < w; ++e) {
              const int64_t g = S.slice_off[s] + 32 * e + lane;
              const int32_t dep = S.col[g];
              if (dep < 0) continue;
              if (split && chunk[dep - R0] != (int32_t)b) {         // an import (DSMEM from the neighbour chunk)
                const int32_t ii = impmap[sweep][b].at(dep - (int32_t)R0);
                const int32_t pslice = imp[sweep][b][ii].second;
                need_pref = std::max(need_pref, sl_lev[sweep][pslice]);
                ent[lane].push_back(Ent{S.val[g], (uint16_t)(R + (upper ? P.imp_L : 0) + ii), false});
                P.near++;
                continue;
              }
              const int32_t pd = upper ? upos[dep - R0] : P.lpos[dep - R0];
              const int32_t q = pd - sb0 * 32;                  // block-relative position
              const bool isnew = sl_lev[sweep][pd / 32] >= (v - lv0) - 1;
              if ((int64_t)send * 32 - 1 - q < R) { ent[lane].push_back(Ent{S.val[g], (uint16_t)(q & (R - 1)), isnew}); P.near++; }
              else { P.far++; }
            }
          }
          if (split) P.sneed.push_back((uint16_t)(need_pref + 1));
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
        }
      }
      P.lev_off.push_back((int32_t)rec);
    }
    P.binfo.insert(P.binfo.end(), info, info + REG_BINFO_INTS);
    P.max_block_slices = std::max(P.max_block_slices, info[1] + info[4]);
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

// Q > 1: the split form (every block's sweeps over a Q-CTA cluster); when it
// cannot be built (a dependency two chunks away, too many imports) the stage
// falls back to Q / 2, down to the one-CTA form.  The split form has no TMA /
// level-kernel variant (their blocks must be independent).
template <typename T>
void pack_stage(const std::vector<int64_t> &blk, const std::vector<Factor<T>> &fac, Stage<T> &S, int Q) {
  S.blk = blk;
  for (; Q > 1; Q /= 2) {
    pack_sweep(blk, fac, false, S.Lp, Q);
    pack_sweep(blk, fac, true, S.Up, Q);
    pack_reg(blk, S.Lp, S.Up, S.reg, Q);
    if (S.reg.ok) {
      S.pipe = PipePack<T>();
      return;
    }
  }
  pack_sweep(blk, fac, false, S.Lp);
  pack_sweep(blk, fac, true, S.Up);
  pack_pipe(blk, S.Lp, S.Up, S.pipe);
  pack_reg(blk, S.Lp, S.Up, S.reg);
}

template void pack_stage<double>(const std::vector<int64_t> &, const std::vector<Factor<double>> &, Stage<double> &, int);
template void pack_stage<zc>(const std::vector<int64_t> &, const std::vector<Factor<zc>> &, Stage<zc> &, int);

}  // namespace gemslr
