// Host stage of setup(A, levels, p, rank): Alg. 1 pGeMSLRSetup lines 1-5
// except the low-rank terms.  Validate A, reorder (Alg. 3), form
// Â = Pᵀ A P, cut it into B_l blocks / E_l / F_l / C_last blocks
// (P:L458-464), factor every block in parallel and
// build the level-scheduled sweeps.
#include <algorithm>
#include <cstring>

#include "plan.hpp"

namespace gemslr {

namespace {

template <typename T>
Csr<T> permute(int64_t n, const int64_t *rowptr, const int32_t *colidx, const T *vals, const Structure &st) {
  Csr<T> B;
  B.n = B.m = n;
  B.ptr.assign(n + 1, 0);
  for (int64_t i = 0; i < n; ++i) {
    const int64_t oi = st.perm[i];
    B.ptr[i + 1] = B.ptr[i] + (rowptr[oi + 1] - rowptr[oi]);
  }
  B.col.resize(B.ptr[n]);
  B.val.resize(B.ptr[n]);
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) {
    const int64_t oi = st.perm[i];
    std::vector<std::pair<int32_t, T>> row;
    row.reserve(rowptr[oi + 1] - rowptr[oi]);
    for (int64_t p = rowptr[oi]; p < rowptr[oi + 1]; ++p) row.push_back({(int32_t)st.iperm[colidx[p]], vals[p]});
    std::sort(row.begin(), row.end(), [](const std::pair<int32_t, T> &a, const std::pair<int32_t, T> &b) { return a.first < b.first; });
    int64_t q = B.ptr[i];
    for (auto &e : row) { B.col[q] = e.first; B.val[q] = e.second; ++q; }
  }
  return B;
}

// A[r0:r1, c0:c1]; rows local (i - r0); columns local (j - c0) when `local_cols`, else absolute.
template <typename T>
Csr<T> sub(const Csr<T> &A, int64_t r0, int64_t r1, int64_t c0, int64_t c1, bool local_cols) {
  Csr<T> S;
  S.n = r1 - r0;
  S.m = local_cols ? c1 - c0 : A.m;
  S.ptr.assign(S.n + 1, 0);
  for (int64_t i = r0; i < r1; ++i) {
    for (int64_t p = A.ptr[i]; p < A.ptr[i + 1]; ++p) {
      const int64_t j = A.col[p];
      if (j >= c0 && j < c1) {
        S.col.push_back((int32_t)(local_cols ? j - c0 : j));
        S.val.push_back(A.val[p]);
      }
    }
    S.ptr[i - r0 + 1] = (int64_t)S.col.size();
  }
  return S;
}

template <typename T>
bool factor_blocks(const Csr<T> &Ahat, const std::vector<int64_t> &bl, const SetupOptions &opt,
                   std::vector<Factor<T>> &out, const std::string &where, Error &err) {
  const int nb = (int)bl.size() - 1;
  out.assign(nb, Factor<T>());
  std::vector<std::string> errs(nb);
  std::vector<char> ok(nb, 1);
#pragma omp parallel for schedule(dynamic, 1)
  for (int q = 0; q < nb; ++q) {
    Csr<T> B = sub(Ahat, bl[q], bl[q + 1], bl[q], bl[q + 1], true);
    ok[q] = opt.ilu == 0 ? ilu0(B, out[q], errs[q]) : ilut(B, opt.tau, opt.lfil, out[q], errs[q]);
  }
  for (int q = 0; q < nb; ++q)
    if (!ok[q]) {
      err = {-4, "ZERO_PIVOT: " + where + ", block " + std::to_string(q) + ": " + errs[q]};
      return false;
    }
  return true;
}

// drop empty blocks for the device stage
template <typename T>
void make_stage(const std::vector<int64_t> &bl, const std::vector<Factor<T>> &fac, Stage<T> &S) {
  std::vector<int64_t> bounds;
  std::vector<Factor<T>> facs;
  for (size_t q = 0; q + 1 < bl.size(); ++q) {
    if (bl[q + 1] == bl[q]) continue;
    if (bounds.empty() || bounds.back() != bl[q]) bounds.push_back(bl[q]);
    bounds.push_back(bl[q + 1]);
    facs.push_back(fac[q]);
  }
  if (bounds.empty()) bounds.push_back(bl.empty() ? 0 : bl[0]);
  pack_stage(bounds, facs, S);
}

}  // namespace

template <typename T>
bool build_host_plan(int64_t n, const int64_t *rowptr, const int32_t *colidx, const T *vals,
                     const SetupOptions &opt, HostPlan<T> &plan, Error &err) {
  // ---- validate CSR: monotone rowptr, columns in range, sorted unique
  if (rowptr[0] != 0) { err = {-2, "BAD_CSR: rowptr[0] != 0"}; return false; }
  for (int64_t i = 0; i < n; ++i) {
    if (rowptr[i + 1] < rowptr[i]) { err = {-2, "BAD_CSR: rowptr not monotone at row " + std::to_string(i)}; return false; }
    for (int64_t p = rowptr[i]; p < rowptr[i + 1]; ++p) {
      if (colidx[p] < 0 || colidx[p] >= n) { err = {-2, "BAD_CSR: column out of range in row " + std::to_string(i)}; return false; }
      if (p > rowptr[i] && colidx[p] <= colidx[p - 1]) { err = {-2, "BAD_CSR: unsorted or duplicate columns in row " + std::to_string(i)}; return false; }
    }
  }
  Graph g = build_graph(n, rowptr, colidx);
  if (!build_structure(g, opt, plan.st, err)) return false;
  const Structure &st = plan.st;
  plan.Ahat = permute(n, rowptr, colidx, vals, st);
  const int L = st.L;
  plan.fac.resize(L);
  plan.E.resize(L);
  plan.F.resize(L);
  plan.stage.resize(L);
  plan.fac_nnz = 0;
  for (int l = 0; l < L; ++l) {
    if (!factor_blocks(plan.Ahat, st.blk[l], opt, plan.fac[l], "level " + std::to_string(l), err)) return false;
    plan.E[l] = sub(plan.Ahat, st.o[l + 1], n, st.o[l], st.o[l + 1], false);
    plan.F[l] = sub(plan.Ahat, st.o[l], st.o[l + 1], st.o[l + 1], n, false);
    for (auto &f : plan.fac[l]) plan.fac_nnz += f.L.nnz() + f.U.nnz();
    make_stage(st.blk[l], plan.fac[l], plan.stage[l]);
  }
  if (!factor_blocks(plan.Ahat, st.last, opt, plan.lastfac, "C_last", err)) return false;
  for (auto &f : plan.lastfac) plan.fac_nnz += f.L.nnz() + f.U.nnz();
  make_stage(st.last, plan.lastfac, plan.last_stage);
  return true;
}

template bool build_host_plan<double>(int64_t, const int64_t *, const int32_t *, const double *,
                                      const SetupOptions &, HostPlan<double> &, Error &);
template bool build_host_plan<zc>(int64_t, const int64_t *, const int32_t *, const zc *,
                                  const SetupOptions &, HostPlan<zc> &, Error &);

}  // namespace gemslr
