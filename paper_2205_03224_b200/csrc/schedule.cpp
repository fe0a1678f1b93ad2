// Level schedules of the triangular substitutions (built once at setup) and
// their SELL-32 packing for the sm_100a trisolve kernel.
//
// Forward sweep (L, unit diagonal): level(i) = 1 + max level(j), j < i in row i
// of L.  Backward sweep (U): level(i) = 1 + max level(j), j > i in row i of U,
// rows taken in descending order.  Rows of one level are independent; inside a
// level they are sorted ascending and packed 32 per slice (one row per lane),
// entries column-major inside the slice so a warp's loads are coalesced.
#include <algorithm>

#include "plan.hpp"

namespace gemslr {

namespace {

template <typename T>
void pack_sweep(const std::vector<int64_t> &blk, const std::vector<Factor<T>> &fac, bool upper, TriPack<T> &P) {
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
    // bucket rows by level (ascending row inside a level)
    std::vector<int64_t> cnt(nlev + 1, 0);
    for (int64_t i = 0; i < n; ++i) cnt[lev[i] + 1]++;
    for (int32_t v = 0; v < nlev; ++v) cnt[v + 1] += cnt[v];
    std::vector<int64_t> rows(n);
    {
      std::vector<int64_t> pos(cnt.begin(), cnt.end() - 1);
      for (int64_t i = 0; i < n; ++i) rows[pos[lev[i]]++] = i;
    }
    for (int32_t v = 0; v < nlev; ++v) {
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

}  // namespace

template <typename T>
void pack_stage(const std::vector<int64_t> &blk, const std::vector<Factor<T>> &fac, Stage<T> &S) {
  S.blk = blk;
  pack_sweep(blk, fac, false, S.Lp);
  pack_sweep(blk, fac, true, S.Up);
}

template void pack_stage<double>(const std::vector<int64_t> &, const std::vector<Factor<double>> &, Stage<double> &);
template void pack_stage<zc>(const std::vector<int64_t> &, const std::vector<Factor<zc>> &, Stage<zc> &);

}  // namespace gemslr
