// Small dense complex Schur decomposition for the thick-restart Arnoldi of
// the low-rank setup ("complex Schur decomposition H_m = Q T Q^H", P:L440;
// P:L393-396).  m <= 2k+2 here, so plain O(m^3) algorithms suffice:
//   Householder reduction to upper Hessenberg form,
//   single-shift (Wilkinson) implicit QR sweeps with deflation,
//   reordering by Givens swaps of adjacent eigenvalues (ztrexc-style).
// Column-major storage, leading dimension n.
#include <cmath>

#include "plan.hpp"

namespace gemslr {

namespace {

inline zc &at(zc *M, int n, int i, int j) { return M[(size_t)j * n + i]; }

// Givens rotation G = [[c, s], [-conj(s), c]] with G [f; g] = [r; 0].
inline void lartg(const zc &f, const zc &g, double &c, zc &s) {
  const double af = std::abs(f), ag = std::abs(g);
  if (ag == 0.0) { c = 1.0; s = 0.0; return; }
  if (af == 0.0) { c = 0.0; s = std::conj(g) / ag; return; }
  const double t = std::hypot(af, ag);
  c = af / t;
  s = (f / af) * std::conj(g) / t;
}

// rows k, k+1 of M (columns j0..n-1) <- G rows
inline void rot_rows(zc *M, int n, int k, int j0, double c, const zc &s) {
  for (int j = j0; j < n; ++j) {
    zc x = at(M, n, k, j), y = at(M, n, k + 1, j);
    at(M, n, k, j) = c * x + s * y;
    at(M, n, k + 1, j) = c * y - std::conj(s) * x;
  }
}
// columns k, k+1 of M (rows 0..i1-1) <- M G^H
inline void rot_cols(zc *M, int ld, int k, int i1, double c, const zc &s) {
  for (int i = 0; i < i1; ++i) {
    zc x = M[(size_t)k * ld + i], y = M[(size_t)(k + 1) * ld + i];
    M[(size_t)k * ld + i] = c * x + std::conj(s) * y;
    M[(size_t)(k + 1) * ld + i] = c * y - s * x;
  }
}

}  // namespace

bool schur_complex(int n, const zc *A, zc *T, zc *Z) {
  for (size_t i = 0; i < (size_t)n * n; ++i) T[i] = A[i];
  for (int j = 0; j < n; ++j)
    for (int i = 0; i < n; ++i) at(Z, n, i, j) = (i == j) ? zc(1) : zc(0);
  // ---- Householder reduction to Hessenberg form
  std::vector<zc> v(n);
  for (int k = 0; k + 2 < n; ++k) {
    double xn = 0;
    for (int i = k + 1; i < n; ++i) xn += abs2(at(T, n, i, k));
    xn = std::sqrt(xn);
    if (xn == 0.0) continue;
    const zc x0 = at(T, n, k + 1, k);
    const zc phase = std::abs(x0) > 0 ? x0 / std::abs(x0) : zc(1);
    for (int i = 0; i < n; ++i) v[i] = 0;
    for (int i = k + 1; i < n; ++i) v[i] = at(T, n, i, k);
    v[k + 1] += phase * xn;
    double vn = 0;
    for (int i = k + 1; i < n; ++i) vn += abs2(v[i]);
    if (vn == 0.0) continue;
    // T <- (I - 2 v v^H / vn) T
    for (int j = 0; j < n; ++j) {
      zc d = 0;
      for (int i = k + 1; i < n; ++i) d += std::conj(v[i]) * at(T, n, i, j);
      d *= 2.0 / vn;
      for (int i = k + 1; i < n; ++i) at(T, n, i, j) -= v[i] * d;
    }
    // T <- T (I - 2 v v^H / vn) ; Z <- Z (I - 2 v v^H / vn)
    for (zc *M : {T, Z}) {
      for (int i = 0; i < n; ++i) {
        zc d = 0;
        for (int j = k + 1; j < n; ++j) d += at(M, n, i, j) * v[j];
        d *= 2.0 / vn;
        for (int j = k + 1; j < n; ++j) at(M, n, i, j) -= d * std::conj(v[j]);
      }
    }
    for (int i = k + 2; i < n; ++i) at(T, n, i, k) = 0;
  }
  // ---- implicit single-shift QR on the Hessenberg matrix
  const double eps = 2.220446049250313e-16;
  double hnorm = 0;
  for (size_t i = 0; i < (size_t)n * n; ++i) hnorm = std::max(hnorm, std::abs(T[i]));
  int hi = n - 1, iter = 0, total = 0;
  while (hi > 0) {
    int l = hi;
    for (; l > 0; --l) {
      double s = std::abs(at(T, n, l - 1, l - 1)) + std::abs(at(T, n, l, l));
      if (s == 0.0) s = hnorm;
      if (std::abs(at(T, n, l, l - 1)) <= eps * s) { at(T, n, l, l - 1) = 0; break; }
    }
    if (l == hi) { --hi; iter = 0; continue; }
    if (++total > 100 * n) return false;
    ++iter;
    zc mu;
    if (iter % 11 == 10) {                                      // exceptional shift
      mu = at(T, n, hi, hi) + zc(std::abs(at(T, n, hi, hi - 1)), 0.0);
    } else {                                                    // Wilkinson shift
      const zc a = at(T, n, hi - 1, hi - 1), b = at(T, n, hi - 1, hi), c = at(T, n, hi, hi - 1), d = at(T, n, hi, hi);
      const zc half = 0.5 * (a - d);
      const zc disc = std::sqrt(half * half + b * c);
      const zc m1 = d - b * c / (half + disc), m2 = d - b * c / (half - disc);
      const bool ok1 = std::abs(half + disc) > 0, ok2 = std::abs(half - disc) > 0;
      if (ok1 && ok2) mu = std::abs(m1 - d) < std::abs(m2 - d) ? m1 : m2;
      else if (ok1) mu = m1;
      else if (ok2) mu = m2;
      else mu = d;
    }
    zc x = at(T, n, l, l) - mu, y = at(T, n, l + 1, l);
    for (int k = l; k < hi; ++k) {
      if (k > l) { x = at(T, n, k, k - 1); y = at(T, n, k + 1, k - 1); }
      double c;
      zc s;
      lartg(x, y, c, s);
      rot_rows(T, n, k, k > l ? k - 1 : l, c, s);
      rot_cols(T, n, k, std::min(k + 3, hi + 1), c, s);
      rot_cols(Z, n, k, n, c, s);
      if (k > l) at(T, n, k + 1, k - 1) = 0;
    }
  }
  for (int j = 0; j < n; ++j)
    for (int i = j + 1; i < n; ++i) at(T, n, i, j) = 0;
  return true;
}

void schur_reorder(int n, zc *T, zc *Z, const std::vector<char> &select) {
  std::vector<char> sel(select);
  int ks = 0;
  for (int j = 0; j < n; ++j) {
    if (!sel[j]) continue;
    for (int k = j - 1; k >= ks; --k) {                         // move position k+1 -> k
      const zc t11 = at(T, n, k, k), t22 = at(T, n, k + 1, k + 1);
      double c;
      zc s;
      lartg(at(T, n, k, k + 1), t22 - t11, c, s);
      if (k + 2 < n) rot_rows(T, n, k, k + 2, c, s);
      rot_cols(T, n, k, k, c, s);
      at(T, n, k, k) = t22;
      at(T, n, k + 1, k + 1) = t11;
      rot_cols(Z, n, k, n, c, s);
      std::swap(sel[k], sel[k + 1]);
    }
    ++ks;
  }
}

}  // namespace gemslr
