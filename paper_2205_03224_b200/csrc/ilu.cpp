// Incomplete LU factorizations of the diagonal blocks B_l^(j) and of the
// C_{l_ev-1} blocks (Alg. 1 lines 3 and 5).
//
// ILU(0): IKJ elimination restricted to the pattern of B.
// ILUT(tau, lfil): Saad's dual-threshold ILU, with the rules of
// reading Q9: tau_i = tau * ||b_i||_2 (squares summed in column
// order), pivots k < i taken in ascending order including fill, a multiplier
// below tau_i is dropped before its update, a second drop of every j != i
// below tau_i, then the lfil largest of L and (separately) of U, ties towards
// the smaller column, diagonal always kept, zero pivot -> error.
// Built with -ffp-contract=off: the arithmetic is IEEE round-to-nearest.
#include <algorithm>
#include <functional>
#include <queue>

#include "plan.hpp"

namespace gemslr {

template <typename T>
bool ilu0(const Csr<T> &B, Factor<T> &F, std::string &err) {
  const int64_t n = B.n;
  std::vector<T> a(B.val);
  std::vector<int64_t> dpos(n, -1), where(n, -1);
  for (int64_t i = 0; i < n; ++i)
    for (int64_t p = B.ptr[i]; p < B.ptr[i + 1]; ++p)
      if (B.col[p] == i) dpos[i] = p;
  for (int64_t i = 0; i < n; ++i) {
    if (dpos[i] < 0) { err = "missing diagonal in row " + std::to_string(i); return false; }
    for (int64_t p = B.ptr[i]; p < B.ptr[i + 1]; ++p) where[B.col[p]] = p;
    for (int64_t p = B.ptr[i]; p < dpos[i]; ++p) {        // k < i, ascending
      const int64_t k = B.col[p];
      a[p] = a[p] / a[dpos[k]];
      const T lik = a[p];
      for (int64_t q = dpos[k] + 1; q < B.ptr[k + 1]; ++q) {
        const int64_t w = where[B.col[q]];
        if (w >= 0) a[w] -= lik * a[q];
      }
    }
    for (int64_t p = B.ptr[i]; p < B.ptr[i + 1]; ++p) where[B.col[p]] = -1;
    if (a[dpos[i]] == T(0)) { err = "zero pivot in row " + std::to_string(i); return false; }
  }
  F = Factor<T>();
  F.L.n = F.L.m = F.U.n = F.U.m = n;
  F.L.ptr.assign(n + 1, 0);
  F.U.ptr.assign(n + 1, 0);
  for (int64_t i = 0; i < n; ++i) {
    for (int64_t p = B.ptr[i]; p < dpos[i]; ++p) { F.L.col.push_back(B.col[p]); F.L.val.push_back(a[p]); }
    for (int64_t p = dpos[i]; p < B.ptr[i + 1]; ++p) { F.U.col.push_back(B.col[p]); F.U.val.push_back(a[p]); }
    F.L.ptr[i + 1] = (int64_t)F.L.col.size();
    F.U.ptr[i + 1] = (int64_t)F.U.col.size();
  }
  return true;
}

template <typename T>
bool ilut(const Csr<T> &B, double tau, int lfil, Factor<T> &F, std::string &err) {
  const int64_t n = B.n;
  F = Factor<T>();
  F.L.n = F.L.m = F.U.n = F.U.m = n;
  F.L.ptr.assign(n + 1, 0);
  F.U.ptr.assign(n + 1, 0);
  std::vector<T> w(n, T(0));
  std::vector<char> inpat(n, 0);
  std::vector<int32_t> pat;
  std::priority_queue<int32_t, std::vector<int32_t>, std::greater<int32_t>> lower;   // pending pivots k < i
  std::vector<std::pair<double, int32_t>> lo, up;
  std::vector<int32_t> sel;
  for (int64_t i = 0; i < n; ++i) {
    pat.clear();
    double nrm2 = 0.0;
    for (int64_t p = B.ptr[i]; p < B.ptr[i + 1]; ++p) {
      const int32_t j = B.col[p];
      w[j] = B.val[p];
      inpat[j] = 1;
      pat.push_back(j);
      nrm2 += abs2(B.val[p]);
      if (j < i) lower.push(j);
    }
    if (!inpat[i]) { w[i] = T(0); inpat[i] = 1; pat.push_back((int32_t)i); }
    const double tau_i = tau * std::sqrt(nrm2);
    while (!lower.empty()) {
      const int32_t k = lower.top();
      lower.pop();
      const int64_t d = F.U.ptr[k];
      w[k] = w[k] / F.U.val[d];
      if (absval(w[k]) < tau_i) { w[k] = T(0); continue; }
      const T wk = w[k];
      for (int64_t q = d + 1; q < F.U.ptr[k + 1]; ++q) {
        const int32_t j = F.U.col[q];
        if (!inpat[j]) {
          inpat[j] = 1;
          w[j] = T(0);
          pat.push_back(j);
          if (j < i) lower.push(j);
        }
        w[j] -= wk * F.U.val[q];
      }
    }
    lo.clear();
    up.clear();
    for (int32_t j : pat) {
      if (j == i) continue;
      const double a = absval(w[j]);
      if (a < tau_i) continue;
      (j < i ? lo : up).push_back({a, j});
    }
    auto larger = [](const std::pair<double, int32_t> &x, const std::pair<double, int32_t> &y) {
      return x.first != y.first ? x.first > y.first : x.second < y.second;
    };
    for (auto *part : {&lo, &up}) {
      if ((int64_t)part->size() > lfil) {
        std::partial_sort(part->begin(), part->begin() + lfil, part->end(), larger);
        part->resize(lfil);
      }
    }
    sel.clear();
    for (auto &e : lo) sel.push_back(e.second);
    std::sort(sel.begin(), sel.end());
    for (int32_t j : sel) { F.L.col.push_back(j); F.L.val.push_back(w[j]); }
    if (w[i] == T(0)) { err = "zero pivot in row " + std::to_string(i); return false; }
    F.U.col.push_back((int32_t)i);
    F.U.val.push_back(w[i]);
    sel.clear();
    for (auto &e : up) sel.push_back(e.second);
    std::sort(sel.begin(), sel.end());
    for (int32_t j : sel) { F.U.col.push_back(j); F.U.val.push_back(w[j]); }
    F.L.ptr[i + 1] = (int64_t)F.L.col.size();
    F.U.ptr[i + 1] = (int64_t)F.U.col.size();
    for (int32_t j : pat) { w[j] = T(0); inpat[j] = 0; }
  }
  return true;
}

template bool ilu0<double>(const Csr<double> &, Factor<double> &, std::string &);
template bool ilu0<zc>(const Csr<zc> &, Factor<zc> &, std::string &);
template bool ilut<double>(const Csr<double> &, double, int, Factor<double> &, std::string &);
template bool ilut<zc>(const Csr<zc> &, double, int, Factor<zc> &, std::string &);

}  // namespace gemslr
