// ============================================================================
// ORACLE — TEST INFRASTRUCTURE ONLY.
//
// A plain, slow, obviously-correct CPU implementation of what the GeMSLR
// solve path computes (arXiv 2205.03224, /root/reference/PAPER.md = "P").
// Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
// --impl reference leg may load this library.  It shares no source with the
// product (paper_2205_03224_b200/csrc) and the product never loads it.
//
// Every function names the passage it follows.  No blocking, fusion or
// reordering beyond what the cited definition/algorithm states.  Compiled
// with -O2 -ffp-contract=off (reading Q22: host-side arithmetic is IEEE
// round-to-nearest with no FMA contraction).
//
//   csr_spmv        y_i = Σ_j a_ij x_j, j ascending          (c2)
//   ilu0            IKJ ILU restricted to the pattern          (Q9)
//   ilut            Saad dual-threshold ILUT(τ, lfil)          (Q9)
//   lsolve/usolve   forward / backward substitution
//   Precond::apply  Alg. 2 pGeMSLRSolve, single-pass, unrolled (c4)
//   Precond::ghat   Ĝ_l = E_l U_l^-1 L_l^-1 F_l C_l^-1        (Q4)
//   fgmres          FGMRES(m) with CGS2 + Givens               (c5; Q14/Q15)
//   fgmres_dcgs2    the same with DCGS2 (lagged reorthogonalisation) (c5'; Q14/Q38)
//
// Pins: see tests/test_oracle_pins.py (closed forms, textbook special cases,
// dense LU/Schur on tiny problems).  Nothing here is "parity unpinned".
//
// Threads: OpenMP only over independent work — rows of a
// SpMV or a vector update, the subdomain blocks of one level (B_l is block
// diagonal), the k columns of W^H z2.  The two reductions over vector entries
// (dot, nrm2) sum fixed chunks of kChunk entries in ascending order and then the
// chunk sums in ascending order, so every result is the same for any thread count.
// ============================================================================
#include <algorithm>
#include <cmath>
#include <complex>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>
#ifdef _OPENMP
#include <omp.h>
#endif

using zc = std::complex<double>;

namespace {

inline double absval(double a) { return std::fabs(a); }
inline double absval(const zc &a) { return std::abs(a); }
inline double abs2(double a) { return a * a; }
inline double abs2(const zc &a) { return a.real() * a.real() + a.imag() * a.imag(); }
inline double conjv(double a) { return a; }
inline zc conjv(const zc &a) { return std::conj(a); }

template <typename T>
struct Csr {
  int64_t n = 0, m = 0;  // rows, cols
  std::vector<int64_t> ptr;
  std::vector<int64_t> col;
  std::vector<T> val;
  int64_t nnz() const { return ptr.empty() ? 0 : ptr[n]; }
};

// ---- c2: plain SpMV, natural order, j ascending ----------------
template <typename T>
void spmv(const Csr<T> &A, const T *x, T *y) {
#pragma omp parallel for schedule(static) if (A.n > 4096)
  for (int64_t i = 0; i < A.n; ++i) {
    T s = T(0);
    for (int64_t p = A.ptr[i]; p < A.ptr[i + 1]; ++p) s += A.val[p] * x[A.col[p]];
    y[i] = s;
  }
}

// y -= A x
template <typename T>
void spmv_sub(const Csr<T> &A, const T *x, T *y) {
#pragma omp parallel for schedule(static) if (A.n > 4096)
  for (int64_t i = 0; i < A.n; ++i) {
    T s = T(0);
    for (int64_t p = A.ptr[i]; p < A.ptr[i + 1]; ++p) s += A.val[p] * x[A.col[p]];
    y[i] -= s;
  }
}

// Submatrix A[r0:r1, c0:c1] with local indices (columns stay sorted).
template <typename T>
Csr<T> submatrix(const Csr<T> &A, int64_t r0, int64_t r1, int64_t c0, int64_t c1) {
  Csr<T> S;
  S.n = r1 - r0;
  S.m = c1 - c0;
  S.ptr.assign(S.n + 1, 0);
  for (int64_t i = r0; i < r1; ++i) {
    for (int64_t p = A.ptr[i]; p < A.ptr[i + 1]; ++p) {
      int64_t j = A.col[p];
      if (j >= c0 && j < c1) {
        S.col.push_back(j - c0);
        S.val.push_back(A.val[p]);
      }
    }
    S.ptr[i - r0 + 1] = (int64_t)S.col.size();
  }
  return S;
}

// ---- ILU factors: L strict-lower (unit diagonal implicit), U upper with the
// diagonal stored first in each row ("A ≈ LU ... two triangular
// substitutions").
template <typename T>
struct Ilu {
  Csr<T> L, U;
};

// ILU(0): IKJ variant restricted to the pattern of B (reading Q9):
// for i; for k < i in pattern(i) ascending: a_ik /= a_kk;
//   for j > k in pattern(k) with (i,j) in pattern: a_ij -= a_ik a_kj.
template <typename T>
Ilu<T> ilu0(const Csr<T> &B, std::string &err) {
  const int64_t n = B.n;
  Csr<T> W = B;  // working copy, rows sorted
  std::vector<int64_t> diagpos(n, -1);
  for (int64_t i = 0; i < n; ++i)
    for (int64_t p = W.ptr[i]; p < W.ptr[i + 1]; ++p)
      if (W.col[p] == i) diagpos[i] = p;
  std::vector<int64_t> where(n, -1);  // column -> position in current row
  for (int64_t i = 0; i < n; ++i) {
    if (diagpos[i] < 0) { err = "ZERO_PIVOT: structurally missing diagonal in row " + std::to_string(i); return {}; }
    for (int64_t p = W.ptr[i]; p < W.ptr[i + 1]; ++p) where[W.col[p]] = p;
    for (int64_t p = W.ptr[i]; p < W.ptr[i + 1]; ++p) {
      int64_t k = W.col[p];
      if (k >= i) break;
      W.val[p] = W.val[p] / W.val[diagpos[k]];
      for (int64_t q = diagpos[k] + 1; q < W.ptr[k + 1]; ++q) {
        int64_t j = W.col[q];
        if (where[j] >= 0) W.val[where[j]] -= W.val[p] * W.val[q];
      }
    }
    for (int64_t p = W.ptr[i]; p < W.ptr[i + 1]; ++p) where[W.col[p]] = -1;
    if (W.val[diagpos[i]] == T(0)) { err = "ZERO_PIVOT in row " + std::to_string(i); return {}; }
  }
  Ilu<T> F;
  F.L.n = F.L.m = F.U.n = F.U.m = n;
  F.L.ptr.assign(n + 1, 0);
  F.U.ptr.assign(n + 1, 0);
  for (int64_t i = 0; i < n; ++i) {
    for (int64_t p = W.ptr[i]; p < W.ptr[i + 1]; ++p)
      if (W.col[p] < i) { F.L.col.push_back(W.col[p]); F.L.val.push_back(W.val[p]); }
    F.U.col.push_back(i);
    F.U.val.push_back(W.val[diagpos[i]]);
    for (int64_t p = W.ptr[i]; p < W.ptr[i + 1]; ++p)
      if (W.col[p] > i) { F.U.col.push_back(W.col[p]); F.U.val.push_back(W.val[p]); }
    F.L.ptr[i + 1] = (int64_t)F.L.col.size();
    F.U.ptr[i + 1] = (int64_t)F.U.col.size();
  }
  return F;
}

// ILUT(τ, lfil): Saad's dual threshold ILU (P:L366-368 cites it; rules = reading Q9):
//  row i: w <- b_i ; τ_i = τ ||b_i||_2 (Σ|b_ij|^2 in ascending column order)
//  for each k < i in the (growing) pattern of w, ascending:
//     w_k <- w_k / u_kk ; if |w_k| < τ_i: w_k <- 0 (dropped, no update)
//     else w_j <- w_j - w_k u_kj for all j > k in row k of U (fill enters the pattern)
//  drop every j != i with |w_j| < τ_i
//  keep the lfil largest |w_j| among j < i and separately among j > i
//  (ties -> smaller j); the diagonal is always kept; u_ii == 0 -> ZERO_PIVOT.
template <typename T>
Ilu<T> ilut(const Csr<T> &B, double tau, int lfil, std::string &err) {
  const int64_t n = B.n;
  Ilu<T> F;
  F.L.n = F.L.m = F.U.n = F.U.m = n;
  F.L.ptr.assign(n + 1, 0);
  F.U.ptr.assign(n + 1, 0);
  std::vector<T> w(n, T(0));
  std::vector<char> in(n, 0);
  std::vector<int64_t> pat;  // pattern of w (unsorted)
  for (int64_t i = 0; i < n; ++i) {
    pat.clear();
    double nrm2 = 0.0;
    for (int64_t p = B.ptr[i]; p < B.ptr[i + 1]; ++p) {
      int64_t j = B.col[p];
      w[j] = B.val[p];
      in[j] = 1;
      pat.push_back(j);
      nrm2 += abs2(B.val[p]);
    }
    if (!in[i]) { w[i] = T(0); in[i] = 1; pat.push_back(i); }
    const double tau_i = tau * std::sqrt(nrm2);
    // eliminate: repeatedly take the smallest k < i not yet processed
    int64_t last = -1;
    while (true) {
      int64_t k = n;
      for (int64_t j : pat)
        if (j > last && j < i && j < k) k = j;
      if (k == n) break;
      last = k;
      // U row k: diagonal first
      const int64_t d = F.U.ptr[k];
      w[k] = w[k] / F.U.val[d];
      if (absval(w[k]) < tau_i) { w[k] = T(0); continue; }
      for (int64_t q = d + 1; q < F.U.ptr[k + 1]; ++q) {
        int64_t j = F.U.col[q];
        if (!in[j]) { in[j] = 1; w[j] = T(0); pat.push_back(j); }
        w[j] -= w[k] * F.U.val[q];
      }
    }
    // second dropping + lfil selection
    std::vector<std::pair<double, int64_t>> lo, up;
    for (int64_t j : pat) {
      if (j == i) continue;
      double a = absval(w[j]);
      if (a < tau_i) continue;
      if (j < i) lo.push_back({a, j}); else up.push_back({a, j});
    }
    auto bigger = [](const std::pair<double, int64_t> &a, const std::pair<double, int64_t> &b) {
      if (a.first != b.first) return a.first > b.first;
      return a.second < b.second;
    };
    std::sort(lo.begin(), lo.end(), bigger);
    std::sort(up.begin(), up.end(), bigger);
    if ((int64_t)lo.size() > lfil) lo.resize(lfil);
    if ((int64_t)up.size() > lfil) up.resize(lfil);
    std::vector<int64_t> lc, uc;
    for (auto &e : lo) lc.push_back(e.second);
    for (auto &e : up) uc.push_back(e.second);
    std::sort(lc.begin(), lc.end());
    std::sort(uc.begin(), uc.end());
    for (int64_t j : lc) { F.L.col.push_back(j); F.L.val.push_back(w[j]); }
    if (w[i] == T(0)) { err = "ZERO_PIVOT in row " + std::to_string(i); return {}; }
    F.U.col.push_back(i);
    F.U.val.push_back(w[i]);
    for (int64_t j : uc) { F.U.col.push_back(j); F.U.val.push_back(w[j]); }
    F.L.ptr[i + 1] = (int64_t)F.L.col.size();
    F.U.ptr[i + 1] = (int64_t)F.U.col.size();
    for (int64_t j : pat) { w[j] = T(0); in[j] = 0; }
  }
  return F;
}

// Forward substitution with unit-lower L: x_i = b_i - Σ_{j<i} l_ij x_j, i ascending.
template <typename T>
void lsolve(const Csr<T> &L, const T *b, T *x) {
  for (int64_t i = 0; i < L.n; ++i) {
    T s = b[i];
    for (int64_t p = L.ptr[i]; p < L.ptr[i + 1]; ++p) s -= L.val[p] * x[L.col[p]];
    x[i] = s;
  }
}
// Backward substitution: x_i = (b_i - Σ_{j>i} u_ij x_j) / u_ii, i descending.
template <typename T>
void usolve(const Csr<T> &U, const T *b, T *x) {
  for (int64_t i = U.n - 1; i >= 0; --i) {
    const int64_t d = U.ptr[i];
    T s = b[i];
    for (int64_t p = d + 1; p < U.ptr[i + 1]; ++p) s -= U.val[p] * x[U.col[p]];
    x[i] = s / U.val[d];
  }
}
template <typename T>
void lusolve(const Ilu<T> &F, const T *b, T *x) {
  std::vector<T> t(F.L.n);
  lsolve(F.L, b, t.data());
  usolve(F.U, t.data(), x);
}

template <typename T>
Ilu<T> factor(const Csr<T> &B, int type, double tau, int lfil, std::string &err) {
  return type == 0 ? ilu0(B, err) : ilut(B, tau, lfil, err);
}

// ---- The GeMSLR preconditioner on a given multilevel structure -------------
// Structure (perm, level offsets, subdomain blocks, C_last blocks) and the
// low-rank terms W_l, G_l are INPUTS (the setup bundle, independently
// verified by tests/); everything else the oracle computes itself from its
// own A: Â = Pᵀ A P, B_l, E_l, F_l (Q3), its own
// ILU factors of every block.
constexpr int64_t kChunk = 8192;           // fixed reduction chunk (thread-count independent)
template <typename T>
T dot(int64_t n, const T *x, const T *y) {  // Σ conj(x_i) y_i (reading Q30)
  const int64_t nc = (n + kChunk - 1) / kChunk;
  std::vector<T> part(nc, T(0));
#pragma omp parallel for schedule(static) if (nc > 1)
  for (int64_t c = 0; c < nc; ++c) {
    T s = T(0);
    for (int64_t i = c * kChunk; i < std::min(n, (c + 1) * kChunk); ++i) s += conjv(x[i]) * y[i];
    part[c] = s;
  }
  T s = T(0);
  for (int64_t c = 0; c < nc; ++c) s += part[c];
  return s;
}
template <typename T>
double nrm2(int64_t n, const T *x) {
  const int64_t nc = (n + kChunk - 1) / kChunk;
  std::vector<double> part(nc, 0.0);
#pragma omp parallel for schedule(static) if (nc > 1)
  for (int64_t c = 0; c < nc; ++c) {
    double s = 0.0;
    for (int64_t i = c * kChunk; i < std::min(n, (c + 1) * kChunk); ++i) s += abs2(x[i]);
    part[c] = s;
  }
  double s = 0.0;
  for (int64_t c = 0; c < nc; ++c) s += part[c];
  return std::sqrt(s);
}

template <typename T>
struct Precond {
  int64_t N = 0;
  int L = 0;
  Csr<T> Ahat;
  std::vector<int64_t> o;                        // o_0..o_L (o_L = start of C_last)
  std::vector<std::vector<int64_t>> blk;         // per level: block boundaries (absolute)
  std::vector<std::vector<Ilu<T>>> fac;          // per level per block
  std::vector<Csr<T>> E, F;                      // E_l: rows J_l, cols I_l ; F_l: rows I_l, cols J_l
  std::vector<int64_t> last;                     // C_last block boundaries (absolute)
  std::vector<Ilu<T>> lastfac;
  std::vector<int> k;                            // rank per level
  std::vector<std::vector<T>> W, G;              // W_l: s_l x k_l col-major; G_l: k_l x k_l col-major

  int64_t s(int l) const { return N - o[l + 1]; }
  int root_its = 0;                              // NEXT-1: inner GMRES steps on Ŝ_0 (0 = single pass)
  Csr<T> C0;                                     // Â[J_0, J_0] (root Schur complement products)

  // rJ += W_l [(I - R_l)^-1 - I] W_l^H rJ   (G_l = (I - R_l)^-1 - I)
  void lowrank_add(int l, T *rJ) const {
    if (k[l] == 0) return;
    const int64_t sl = s(l);
    const int kl = k[l];
    std::vector<T> sv(kl, T(0)), tv(kl, T(0));
#pragma omp parallel for schedule(static)
    for (int c = 0; c < kl; ++c) {                 // s = W^H z2
      T acc = T(0);
      for (int64_t i = 0; i < sl; ++i) acc += conjv(W[l][c * sl + i]) * rJ[i];
      sv[c] = acc;
    }
    for (int a = 0; a < kl; ++a) {                 // t = G s
      T acc = T(0);
      for (int c = 0; c < kl; ++c) acc += G[l][c * kl + a] * sv[c];
      tv[a] = acc;
    }
#pragma omp parallel for schedule(static) if (sl > 4096)
    for (int64_t i = 0; i < sl; ++i) {             // z2 += W t
      T acc = T(0);
      for (int c = 0; c < kl; ++c) acc += W[l][c * sl + i] * tv[c];
      rJ[i] += acc;
    }
  }

  // B_l^{-1} approximated blockwise: x[I_l] = U^-1 L^-1 b[I_l] per block
  void block_solve(int l, const T *b, T *x) const {
    const int64_t nb = (int64_t)blk[l].size() - 1;
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t q = 0; q < nb; ++q) {
      const int64_t a = blk[l][q] - o[l];
      lusolve(fac[l][q], b + a, x + a);
    }
  }
  // C_{L-1}^{-1} by block-Jacobi ILU of the RCM-ordered last separator
  void last_solve(const T *b, T *x) const {
    const int64_t nb = (int64_t)last.size() - 1;
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t q = 0; q < nb; ++q) {
      const int64_t a = last[q] - o[L];
      lusolve(lastfac[q], b + a, x + a);
    }
  }

  // Alg. 2, single-pass reading Q2, unrolled into a down and an
  // up sweep (c4).  Applies C_{l0-1}^{-1}: input r and output y live on
  // positions [o_{l0}, N) (l0 = 0 is the whole preconditioner M^{-1}).
  void apply_from(int l0, const T *r_in, T *y_out) const {
    if (l0 == 0 && root_its > 0) { apply_root(r_in, y_out); return; }
    const int64_t base = o[l0];
    const int64_t n = N - base;
    std::vector<T> r(r_in, r_in + n);
    std::vector<std::vector<T>> z(L);
    for (int l = l0; l < L; ++l) {                     // Alg. 2 lines 2-8, going down
      const int64_t nI = o[l + 1] - o[l];
      T *rI = r.data() + (o[l] - base);
      T *rJ = r.data() + (o[l + 1] - base);
      z[l].assign(nI, T(0));
      block_solve(l, rI, z[l].data());                 // z1 = U_l^-1 L_l^-1 b1
      spmv_sub(E[l], z[l].data(), rJ);                 // z2 = b2 - E_l z1
      if (k[l] > 0) {                                  // u2 + z2, u2 = W[(I-R)^-1 - I]W^H z2
        const int64_t sl = s(l);
        const int kl = k[l];
        std::vector<T> sv(kl, T(0)), tv(kl, T(0));
#pragma omp parallel for schedule(static)
        for (int c = 0; c < kl; ++c) {                 // s = W^H z2
          T acc = T(0);
          for (int64_t i = 0; i < sl; ++i) acc += conjv(W[l][c * sl + i]) * rJ[i];
          sv[c] = acc;
        }
        for (int a = 0; a < kl; ++a) {                 // t = G s, G = (I-R)^-1 - I
          T acc = T(0);
          for (int c = 0; c < kl; ++c) acc += G[l][c * kl + a] * sv[c];
          tv[a] = acc;
        }
#pragma omp parallel for schedule(static) if (sl > 4096)
        for (int64_t i = 0; i < sl; ++i) {             // z2 += W t
          T acc = T(0);
          for (int c = 0; c < kl; ++c) acc += W[l][c * sl + i] * tv[c];
          rJ[i] += acc;
        }
      }
    }
    std::vector<T> y(n, T(0));
    last_solve(r.data() + (o[L] - base), y.data() + (o[L] - base));   // recursion bottom
    for (int l = L - 1; l >= l0; --l) {                // Alg. 2 line 9, coming up
      const int64_t nI = o[l + 1] - o[l];
      T *yI = y.data() + (o[l] - base);
      const T *yJ = y.data() + (o[l + 1] - base);
      std::vector<T> t(nI, T(0)), w(nI, T(0));
      spmv(F[l], yJ, t.data());                        // F_l y2
      block_solve(l, t.data(), w.data());              // U^-1 L^-1 F_l y2
#pragma omp parallel for schedule(static) if (nI > 4096)
      for (int64_t i = 0; i < nI; ++i) yI[i] = z[l][i] - w[i];   // y1 = z1 - ...
    }
    std::copy(y.begin(), y.end(), y_out);
  }

  // ---- NEXT-1: Alg. 2 at the root level with "right preconditioned GMRES" on
  // the inexact Schur complement Ŝ_0 = C_0 - E_0 U_0^-1 L_0^-1 F_0 (P:L541-545,
  // P:L557): z1 = U^-1 L^-1 b1; z2 = b2 - E_0 z1; y2 ≈ Ŝ_0^-1 z2 by root_its
  // steps of GMRES right-preconditioned by P(v) = C_0^-1 (v + W_0 G_0 W_0^H v)
  // (the rank-k branch of Alg. 2 lines 7-8 applied at l = 0; reading Q34);
  // y1 = z1 - U^-1 L^-1 F_0 y2.
  void schur0(const T *v, T *out) const {        // Ŝ_0 v
    const int64_t nI = o[1] - o[0];
    std::vector<T> t(nI, T(0)), u(nI, T(0));
    spmv(C0, v, out);                            // C_0 v
    spmv(F[0], v, t.data());
    block_solve(0, t.data(), u.data());
    spmv_sub(E[0], u.data(), out);               // - E_0 U^-1 L^-1 F_0 v
  }
  void prec0(const T *v, T *out) const {         // P(v) = C_0^-1 (v + W_0 G_0 W_0^H v)
    std::vector<T> u(v, v + s(0));
    lowrank_add(0, u.data());
    apply_from(1, u.data(), out);
  }
  // GMRES(root_its), x0 = 0, right-preconditioned in the flexible form
  // (x = Z y with Z_j = P(V_j)), CGS2 and Givens exactly as the outer c5; it
  // stops early only on breakdown (h_{j+1,j} <= 1e-14 ||w before GS||).
  void root_gmres(const T *b, T *x) const {
    const int64_t n = s(0);
    const int m = root_its;
    std::fill(x, x + n, T(0));
    const double beta = nrm2(n, b);
    if (beta == 0.0) return;
    std::vector<T> V((size_t)n * (m + 1)), Z((size_t)n * m), w(n), H((size_t)(m + 1) * m, T(0)), g(m + 1, T(0));
    std::vector<double> cs(m);
    std::vector<T> sn(m);
    for (int64_t i = 0; i < n; ++i) V[i] = b[i] / beta;
    g[0] = beta;
    int jend = 0;
    for (int j = 0; j < m; ++j) {
      T *vj = V.data() + (size_t)j * n, *zj = Z.data() + (size_t)j * n;
      prec0(vj, zj);
      schur0(zj, w.data());
      const double eta = nrm2(n, w.data());
      std::vector<T> h(j + 1), h2(j + 1);
      for (int i = 0; i <= j; ++i) h[i] = dot(n, V.data() + (size_t)i * n, w.data());
      for (int i = 0; i <= j; ++i)
        for (int64_t q = 0; q < n; ++q) w[q] -= V[(size_t)i * n + q] * h[i];
      for (int i = 0; i <= j; ++i) h2[i] = dot(n, V.data() + (size_t)i * n, w.data());
      for (int i = 0; i <= j; ++i)
        for (int64_t q = 0; q < n; ++q) w[q] -= V[(size_t)i * n + q] * h2[i];
      const double hnext = nrm2(n, w.data());
      T *Hj = H.data() + (size_t)j * (m + 1);
      for (int i = 0; i <= j; ++i) Hj[i] = h[i] + h2[i];
      Hj[j + 1] = hnext;
      for (int i = 0; i < j; ++i) {
        T p = Hj[i], q = Hj[i + 1];
        Hj[i] = cs[i] * p + conjv(sn[i]) * q;
        Hj[i + 1] = -sn[i] * p + cs[i] * q;
      }
      T a = Hj[j];
      double bb = absval(Hj[j + 1]), aa = absval(a), c;
      T sr;
      if (bb == 0.0) { c = 1.0; sr = T(0); }
      else if (aa == 0.0) { c = 0.0; sr = T(1); }
      else {
        double t = std::sqrt(aa * aa + bb * bb);
        c = aa / t;
        sr = bb * conjv(a) / (aa * t);
      }
      cs[j] = c; sn[j] = sr;
      T p = Hj[j], q = Hj[j + 1];
      Hj[j] = c * p + conjv(sr) * q;
      Hj[j + 1] = -sr * p + c * q;
      T gp = g[j], gq = g[j + 1];
      g[j] = c * gp + conjv(sr) * gq;
      g[j + 1] = -sr * gp + c * gq;
      jend = j + 1;
      if (hnext <= 1e-14 * eta) break;
      for (int64_t q2 = 0; q2 < n; ++q2) V[(size_t)(j + 1) * n + q2] = w[q2] / hnext;
    }
    std::vector<T> y(jend);
    for (int i = jend - 1; i >= 0; --i) {          // H[0:jend, 0:jend] y = g
      T acc = g[i];
      for (int c2 = i + 1; c2 < jend; ++c2) acc -= H[(size_t)c2 * (m + 1) + i] * y[c2];
      y[i] = acc / H[(size_t)i * (m + 1) + i];
    }
    for (int c2 = 0; c2 < jend; ++c2)              // x = Z y
      for (int64_t i = 0; i < n; ++i) x[i] += Z[(size_t)c2 * n + i] * y[c2];
  }
  void apply_root(const T *r, T *y) const {
    const int64_t nI = o[1] - o[0], n0 = s(0);
    std::vector<T> z1(nI, T(0)), z2(r + nI, r + nI + n0), y2(n0), t(nI, T(0)), w(nI, T(0));
    block_solve(0, r, z1.data());                  // z1 = U^-1 L^-1 b1
    spmv_sub(E[0], z1.data(), z2.data());          // z2 = b2 - E_0 z1
    root_gmres(z2.data(), y2.data());              // y2 ≈ Ŝ_0^-1 z2
    spmv(F[0], y2.data(), t.data());
    block_solve(0, t.data(), w.data());
    for (int64_t i = 0; i < nI; ++i) y[i] = z1[i] - w[i];   // y1 = z1 - U^-1 L^-1 F_0 y2
    std::copy(y2.begin(), y2.end(), y + nI);
  }

  // Ĝ_l v = E_l (L_l U_l)^{-1} F_l C_l^{-1} v   (Q4)
  void ghat(int l, const T *v, T *out) const {
    const int64_t sl = s(l), nI = o[l + 1] - o[l];
    std::vector<T> c(sl), t(nI), u(nI);
    apply_from(l + 1, v, c.data());
    spmv(F[l], c.data(), t.data());
    block_solve(l, t.data(), u.data());
    spmv(E[l], u.data(), out);
  }
};

// ---- c5: FGMRES(m) with CGS2 (Q14, Q15) ------------------------
typedef void (*precond_fn)(void *user, const void *in, void *out);

template <typename T>
struct FgmresOut {
  int its = 0;
  std::vector<double> hist;
  double final_relres = 0.0;
  int status = 0;
  double max_orth = 0.0;       // max over cycles of ||V^H V - I||_max (diagnostic)
  double max_arnoldi = 0.0;    // max over cycles of ||A Z_j - V_{j+1} Hbar_j||_F / (||A||_F ||Z_j||_F)
  double max_est_gap = 0.0;    // max |estimate - explicit| / bnorm at cycle ends
};


template <typename T>
FgmresOut<T> fgmres(const Csr<T> &A, precond_fn M, void *Muser, const T *b, T *x,
                    double rtol, int m, int maxit, bool diag) {
  const int64_t n = A.n;
  FgmresOut<T> out;
  const double bnorm = nrm2(n, b);
  if (bnorm == 0.0) {
    std::fill(x, x + n, T(0));
    out.hist.push_back(0.0);
    return out;
  }
  double afro = 0.0;
  for (int64_t p = 0; p < A.nnz(); ++p) afro += abs2(A.val[p]);
  afro = std::sqrt(afro);
  std::vector<T> r(n), w(n), V((size_t)n * (m + 1)), Z((size_t)n * m);
  std::vector<T> H((size_t)(m + 1) * m), Hraw((size_t)(m + 1) * m), g(m + 1);
  std::vector<double> cs(m);
  std::vector<T> sn(m);
  auto resid = [&]() {                                      // r = b - A x
    spmv(A, x, r.data());
#pragma omp parallel for schedule(static) if (n > 4096)
    for (int64_t i = 0; i < n; ++i) r[i] = b[i] - r[i];
    return nrm2(n, r.data());
  };
  double beta = resid();
  out.hist.push_back(beta / bnorm);
  while (beta > rtol * bnorm && out.its < maxit) {
#pragma omp parallel for schedule(static) if (n > 4096)
    for (int64_t i = 0; i < n; ++i) V[i] = r[i] / beta;
    std::fill(g.begin(), g.end(), T(0));
    std::fill(H.begin(), H.end(), T(0));
    std::fill(Hraw.begin(), Hraw.end(), T(0));
    g[0] = beta;
    int jend = 0;
    for (int j = 0; j < m; ++j) {
      T *vj = V.data() + (size_t)j * n;
      T *zj = Z.data() + (size_t)j * n;
      if (M) M(Muser, vj, zj); else std::copy(vj, vj + n, zj);   // Z_j = M(V_j)
      spmv(A, zj, w.data());                                      // w = A Z_j
      const double eta = nrm2(n, w.data());
      std::vector<T> h(j + 1), h2(j + 1);
      for (int i = 0; i <= j; ++i) h[i] = dot(n, V.data() + (size_t)i * n, w.data());   // pass 1
#pragma omp parallel for schedule(static) if (n > 4096)
      for (int64_t q = 0; q < n; ++q)                       // w -= V h (per entry, i ascending)
        for (int i = 0; i <= j; ++i) w[q] -= V[(size_t)i * n + q] * h[i];
      for (int i = 0; i <= j; ++i) h2[i] = dot(n, V.data() + (size_t)i * n, w.data());  // pass 2
#pragma omp parallel for schedule(static) if (n > 4096)
      for (int64_t q = 0; q < n; ++q)                       // w -= V h2
        for (int i = 0; i <= j; ++i) w[q] -= V[(size_t)i * n + q] * h2[i];
      const double hnext = nrm2(n, w.data());
      for (int i = 0; i <= j; ++i) H[(size_t)j * (m + 1) + i] = h[i] + h2[i];
      H[(size_t)j * (m + 1) + j + 1] = hnext;
      for (int i = 0; i <= j + 1; ++i) Hraw[(size_t)j * (m + 1) + i] = H[(size_t)j * (m + 1) + i];
      T *Hj = H.data() + (size_t)j * (m + 1);
      for (int i = 0; i < j; ++i) {                         // previous rotations
        T p = Hj[i], q = Hj[i + 1];
        Hj[i] = cs[i] * p + conjv(sn[i]) * q;
        Hj[i + 1] = -sn[i] * p + cs[i] * q;
      }
      {                                                     // rotation j
        T a = Hj[j];
        double bb = absval(Hj[j + 1]);
        double aa = absval(a);
        double c; T s;
        if (bb == 0.0) { c = 1.0; s = T(0); }
        else if (aa == 0.0) { c = 0.0; s = T(1); }
        else {
          double t = std::sqrt(aa * aa + bb * bb);
          c = aa / t;
          s = bb * conjv(a) / (aa * t);
        }
        cs[j] = c; sn[j] = s;
        T p = Hj[j], q = Hj[j + 1];
        Hj[j] = c * p + conjv(s) * q;
        Hj[j + 1] = -s * p + c * q;
        T gp = g[j], gq = g[j + 1];
        g[j] = c * gp + conjv(s) * gq;
        g[j + 1] = -s * gp + c * gq;
      }
      out.its += 1;
      out.hist.push_back(absval(g[j + 1]) / bnorm);
      jend = j + 1;
      if (absval(g[j + 1]) <= rtol * bnorm || hnext <= 1e-14 * eta || out.its >= maxit) break;
      T *vn = V.data() + (size_t)(j + 1) * n;
#pragma omp parallel for schedule(static) if (n > 4096)
      for (int64_t q = 0; q < n; ++q) vn[q] = w[q] / hnext;
    }
    if (diag) {
      // orthonormality of V_0..V_{jend-1}
      for (int a = 0; a < jend; ++a)
        for (int c = 0; c < jend; ++c) {
          T d = dot(n, V.data() + (size_t)a * n, V.data() + (size_t)c * n);
          double e = absval(d - (a == c ? T(1) : T(0)));
          out.max_orth = std::max(out.max_orth, e);
        }
      // Arnoldi relation A Z_c = Σ_{i<=c+1} V_i Hbar_{i,c} for the columns c whose
      // v_{c+1} was formed (the breaking iteration leaves v_{jend} unformed).
      const int ncheck = jend - 1;
      if (ncheck > 0) {
        double num = 0.0, zf = 0.0;
        for (int c = 0; c < ncheck; ++c) {
          const T *zc = Z.data() + (size_t)c * n;
          spmv(A, zc, w.data());
          for (int i = 0; i <= c + 1; ++i) {
            const T *vi = V.data() + (size_t)i * n;
            for (int64_t q = 0; q < n; ++q) w[q] -= vi[q] * Hraw[(size_t)c * (m + 1) + i];
          }
          num += abs2(nrm2(n, w.data()));
          zf += abs2(nrm2(n, zc));
        }
        out.max_arnoldi = std::max(out.max_arnoldi, std::sqrt(num) / (afro * std::sqrt(zf)));
      }
    }
    // y = H[0:jend,0:jend]^{-1} g[0:jend] (upper triangular after the rotations)
    std::vector<T> y(jend);
    for (int i = jend - 1; i >= 0; --i) {
      T s = g[i];
      for (int c = i + 1; c < jend; ++c) s -= H[(size_t)c * (m + 1) + i] * y[c];
      y[i] = s / H[(size_t)i * (m + 1) + i];
    }
#pragma omp parallel for schedule(static) if (n > 4096)
    for (int64_t q = 0; q < n; ++q)                          // x += Z y (per entry, c ascending)
      for (int c = 0; c < jend; ++c) x[q] += Z[(size_t)c * n + q] * y[c];
    const double est = out.hist.back();
    beta = resid();                                          // explicit residual
    out.max_est_gap = std::max(out.max_est_gap, std::fabs(est - beta / bnorm));
  }
  out.final_relres = beta / bnorm;
  out.status = (beta > rtol * bnorm) ? 1 : 0;
  return out;
}

// ---- c5': FGMRES(m) with DCGS2 (reading Q38; Q14 admits a lagged variant when
// both sides adopt it) ----------------------------------------------------------
// Classical Gram-Schmidt applied twice, as CGS2, but the second projection of the
// vector made at step j, and its normalisation, are delayed to step j + 1, where
// they share the passes over the basis with step j + 1's first projection
// (Swirydowicz, Langou, Ananthan, Yang, Thomas, "Low synchronization Gram-Schmidt
// and GMRES algorithms", DCGS2-Arnoldi).  u_j is the not yet reorthogonalised,
// unnormalised new vector (u_0 = r).  Step j:
//   z_j = M(u_j) ; w = A z_j
//   c = V_{0:j}^H u_j ; nu = u_j^H u_j ; a = V_{0:j}^H w ; mu = u_j^H w ; eta = ||w||
//   alpha = sqrt(max(nu - ||c||^2, 0))                       (Pythagoras)
//   column j-1 completed: Hraw[0:j, j-1] += c, Hraw[j, j-1] = alpha   (j = 0: g_0 = alpha)
//   h_j = (mu - c^H a) / alpha
//   v_j = (u_j - V_{0:j} c) / alpha
//   u_{j+1} = w - V_{0:j} a - v_j h_j ; beta_j = ||u_{j+1}||
//   Hraw[0:j, j] = a, Hraw[j, j] = h_j                       (completed at step j + 1)
//   the cycle ends after step j when the residual estimate with H[j+1, j] = beta_j
//   meets rtol, beta_j <= 1e-14 eta (breakdown), its reaches maxit, or j + 1 = m;
//   then one more dot pass (c = V_{0:jend}^H u_jend, nu) completes the last column.
// Each completed column gets the Givens rotations of c5 and one history entry.
template <typename T>
FgmresOut<T> fgmres_dcgs2(const Csr<T> &A, precond_fn M, void *Muser, const T *b, T *x,
                          double rtol, int m, int maxit, bool diag) {
  const int64_t n = A.n;
  FgmresOut<T> out;
  const double bnorm = nrm2(n, b);
  if (bnorm == 0.0) {
    std::fill(x, x + n, T(0));
    out.hist.push_back(0.0);
    return out;
  }
  double afro = 0.0;
  for (int64_t p = 0; p < A.nnz(); ++p) afro += abs2(A.val[p]);
  afro = std::sqrt(afro);
  std::vector<T> r(n), w(n), V((size_t)n * (m + 1)), Z((size_t)n * m);
  std::vector<T> H((size_t)(m + 1) * m), Hraw((size_t)(m + 1) * m), g(m + 1);
  std::vector<double> cs(m);
  std::vector<T> sn(m);
  auto resid = [&]() {                                      // r = b - A x
    spmv(A, x, r.data());
#pragma omp parallel for schedule(static) if (n > 4096)
    for (int64_t i = 0; i < n; ++i) r[i] = b[i] - r[i];
    return nrm2(n, r.data());
  };
  auto col = [&](std::vector<T> &M_, int j) { return M_.data() + (size_t)j * (m + 1); };
  // Givens rotations of c5 on the completed column j (Hraw -> H), then rotation j
  auto finish_column = [&](int j) {
    T *Hj = col(H, j);
    for (int i = 0; i <= j + 1; ++i) Hj[i] = col(Hraw, j)[i];
    for (int i = 0; i < j; ++i) {
      T p = Hj[i], q = Hj[i + 1];
      Hj[i] = cs[i] * p + conjv(sn[i]) * q;
      Hj[i + 1] = -sn[i] * p + cs[i] * q;
    }
    T a = Hj[j];
    double bb = absval(Hj[j + 1]);
    double aa = absval(a);
    double c; T s;
    if (bb == 0.0) { c = 1.0; s = T(0); }
    else if (aa == 0.0) { c = 0.0; s = T(1); }
    else {
      double t = std::sqrt(aa * aa + bb * bb);
      c = aa / t;
      s = bb * conjv(a) / (aa * t);
    }
    cs[j] = c; sn[j] = s;
    T p = Hj[j], q = Hj[j + 1];
    Hj[j] = c * p + conjv(s) * q;
    Hj[j + 1] = -s * p + c * q;
    T gp = g[j], gq = g[j + 1];
    g[j] = c * gp + conjv(s) * gq;
    g[j + 1] = -s * gp + c * gq;
    out.its += 1;
    out.hist.push_back(absval(g[j + 1]) / bnorm);
  };
  // c = V_{0:j}^H u_j, nu = u_j^H u_j, alpha (u_j in column j of V)
  auto reorth_coeffs = [&](int j, std::vector<T> &c, double &alpha) {
    const T *u = V.data() + (size_t)j * n;
    c.assign(j, T(0));
    for (int i = 0; i < j; ++i) c[i] = dot(n, V.data() + (size_t)i * n, u);
    const double nu = abs2(nrm2(n, u));
    double cc = 0.0;
    for (int i = 0; i < j; ++i) cc += abs2(c[i]);
    alpha = std::sqrt(std::max(nu - cc, 0.0));
  };
  auto complete = [&](int j, const std::vector<T> &c, double alpha) {   // column j - 1 (j >= 1)
    T *Hr = col(Hraw, j - 1);
    for (int i = 0; i < j; ++i) Hr[i] += c[i];
    Hr[j] = alpha;
    finish_column(j - 1);
  };
  double beta = resid();
  out.hist.push_back(beta / bnorm);
  while (beta > rtol * bnorm && out.its < maxit) {
    std::copy(r.begin(), r.end(), V.begin());                // u_0 = r
    std::fill(g.begin(), g.end(), T(0));
    std::fill(H.begin(), H.end(), T(0));
    std::fill(Hraw.begin(), Hraw.end(), T(0));
    int jend = 0;
    for (int j = 0; j < m; ++j) {
      T *uj = V.data() + (size_t)j * n;
      T *zj = Z.data() + (size_t)j * n;
      if (M) M(Muser, uj, zj); else std::copy(uj, uj + n, zj);   // z_j = M(u_j)
      spmv(A, zj, w.data());                                      // w = A z_j
      std::vector<T> c, a(j);
      double alpha;
      reorth_coeffs(j, c, alpha);                                 // the dots of the step's one pass
      for (int i = 0; i < j; ++i) a[i] = dot(n, V.data() + (size_t)i * n, w.data());
      const T mu = dot(n, uj, w.data());
      const double eta = nrm2(n, w.data());
      if (j == 0) g[0] = alpha;                                   // r = alpha v_0
      else complete(j, c, alpha);
      T ca = T(0);
      for (int i = 0; i < j; ++i) ca += conjv(c[i]) * a[i];
      const T hj = (mu - ca) / alpha;
      T *un = V.data() + (size_t)(j + 1) * n;
#pragma omp parallel for schedule(static) if (n > 4096)
      for (int64_t q = 0; q < n; ++q) {                      // v_j, then u_{j+1} (per entry, i ascending)
        T v = uj[q];
        for (int i = 0; i < j; ++i) v -= V[(size_t)i * n + q] * c[i];
        v = v / alpha;
        T t = w[q];
        for (int i = 0; i < j; ++i) t -= V[(size_t)i * n + q] * a[i];
        t -= v * hj;
        uj[q] = v;
        un[q] = t;
      }
      const double bj = nrm2(n, un);
      T *Hr = col(Hraw, j);
      for (int i = 0; i < j; ++i) Hr[i] = a[i];
      Hr[j] = hj;
      // the estimate after column j with H[j+1, j] = beta_j (rotations 0..j-1 are final)
      std::vector<T> t(Hr, Hr + j + 1);
      for (int i = 0; i < j; ++i) {
        T p = t[i], q = t[i + 1];
        t[i] = cs[i] * p + conjv(sn[i]) * q;
        t[i + 1] = -sn[i] * p + cs[i] * q;
      }
      const double tt = std::sqrt(abs2(t[j]) + bj * bj);
      const double est = tt > 0.0 ? absval(g[j]) * bj / tt : absval(g[j]);
      jend = j + 1;
      if (est <= rtol * bnorm || bj <= 1e-14 * eta || out.its + 1 >= maxit) break;
    }
    {                                                         // complete column jend - 1
      std::vector<T> c;
      double alpha;
      reorth_coeffs(jend, c, alpha);
      complete(jend, c, alpha);
    }
    if (diag) {
      for (int a = 0; a < jend; ++a)
        for (int c = 0; c < jend; ++c) {
          T d = dot(n, V.data() + (size_t)a * n, V.data() + (size_t)c * n);
          out.max_orth = std::max(out.max_orth, absval(d - (a == c ? T(1) : T(0))));
        }
      // A Z_c = Σ_{i<=c+1} V_i Hraw_{i,c} for c < jend - 1 (v_{jend} is never formed)
      const int ncheck = jend - 1;
      if (ncheck > 0) {
        double num = 0.0, zf = 0.0;
        for (int c = 0; c < ncheck; ++c) {
          const T *zc = Z.data() + (size_t)c * n;
          spmv(A, zc, w.data());
          for (int i = 0; i <= c + 1; ++i) {
            const T *vi = V.data() + (size_t)i * n;
            for (int64_t q = 0; q < n; ++q) w[q] -= vi[q] * Hraw[(size_t)c * (m + 1) + i];
          }
          num += abs2(nrm2(n, w.data()));
          zf += abs2(nrm2(n, zc));
        }
        out.max_arnoldi = std::max(out.max_arnoldi, std::sqrt(num) / (afro * std::sqrt(zf)));
      }
    }
    std::vector<T> y(jend);                                  // y = H^-1 g (c5)
    for (int i = jend - 1; i >= 0; --i) {
      T s = g[i];
      for (int c = i + 1; c < jend; ++c) s -= H[(size_t)c * (m + 1) + i] * y[c];
      y[i] = s / H[(size_t)i * (m + 1) + i];
    }
#pragma omp parallel for schedule(static) if (n > 4096)
    for (int64_t q = 0; q < n; ++q)
      for (int c = 0; c < jend; ++c) x[q] += Z[(size_t)c * n + q] * y[c];
    const double est = out.hist.back();
    beta = resid();
    out.max_est_gap = std::max(out.max_est_gap, std::fabs(est - beta / bnorm));
  }
  out.final_relres = beta / bnorm;
  out.status = (beta > rtol * bnorm) ? 1 : 0;
  return out;
}

template <typename T>
Csr<T> make_csr(int64_t n, const int64_t *rowptr, const int32_t *col, const void *val) {
  Csr<T> A;
  A.n = A.m = n;
  A.ptr.assign(rowptr, rowptr + n + 1);
  A.col.assign(col, col + rowptr[n]);
  const T *v = static_cast<const T *>(val);
  A.val.assign(v, v + rowptr[n]);
  return A;
}

// Â = Pᵀ A P with perm[new] = old: Â[i,j] = A[perm[i], perm[j]].
template <typename T>
Csr<T> permute(const Csr<T> &A, const int64_t *perm) {
  const int64_t n = A.n;
  std::vector<int64_t> iperm(n);
  for (int64_t i = 0; i < n; ++i) iperm[perm[i]] = i;
  Csr<T> B;
  B.n = B.m = n;
  B.ptr.assign(n + 1, 0);
  B.col.reserve(A.nnz());
  B.val.reserve(A.nnz());
  std::vector<std::pair<int64_t, T>> row;
  for (int64_t i = 0; i < n; ++i) {
    const int64_t oi = perm[i];
    row.clear();
    for (int64_t p = A.ptr[oi]; p < A.ptr[oi + 1]; ++p) row.push_back({iperm[A.col[p]], A.val[p]});
    std::sort(row.begin(), row.end(), [](const std::pair<int64_t, T> &a, const std::pair<int64_t, T> &b) { return a.first < b.first; });
    for (auto &e : row) { B.col.push_back(e.first); B.val.push_back(e.second); }
    B.ptr[i + 1] = (int64_t)B.col.size();
  }
  return B;
}

// Complex diagonal shift of the ILU factorizations: "a complex
// shift equal to 0.05 i Σ_i |A_ii| / n_A during the ILU factorization of the
// on-diagonal blocks" — sigma = i * factor * Σ|a_ii| / n, added to the diagonal
// of every block before it is factored (reading Q33: B_l blocks and the C_last
// blocks; complex problems only).
template <typename T> T shift_sigma(const Csr<T> &, double) { return T(0); }
template <> zc shift_sigma<zc>(const Csr<zc> &A, double factor) {
  if (factor == 0.0) return zc(0);
  double s = 0;
  for (int64_t i = 0; i < A.n; ++i)
    for (int64_t p = A.ptr[i]; p < A.ptr[i + 1]; ++p)
      if (A.col[p] == i) s += std::abs(A.val[p]);
  return zc(0.0, factor * s / (double)A.n);
}
template <typename T>
void add_diag(Csr<T> &B, T sigma) {
  for (int64_t i = 0; i < B.n; ++i)
    for (int64_t p = B.ptr[i]; p < B.ptr[i + 1]; ++p)
      if (B.col[p] == i) B.val[p] += sigma;
}

template <typename T>
Precond<T> *build_precond(int64_t n, const int64_t *rowptr, const int32_t *col, const void *val,
                          const int64_t *perm, int L, const int64_t *level_off,
                          const int32_t *nblk, const int64_t *blk_off, int nlast, const int64_t *last_off,
                          int ilu_type, double tau, int lfil, double shift, std::string &err) {
  Csr<T> A = make_csr<T>(n, rowptr, col, val);
  const T sigma = shift_sigma<T>(A, shift);
  auto *P = new Precond<T>();
  P->N = n;
  P->L = L;
  P->Ahat = permute(A, perm);
  P->o.assign(level_off, level_off + L + 1);
  P->k.assign(L, 0);
  P->W.resize(L);
  P->G.resize(L);
  size_t pos = 0;
  for (int l = 0; l < L; ++l) {
    std::vector<int64_t> b(blk_off + pos, blk_off + pos + nblk[l] + 1);
    pos += nblk[l] + 1;
    P->blk.push_back(b);
    std::vector<Ilu<T>> f(nblk[l]);                // blocks of B_l are independent
    std::vector<std::string> errs(nblk[l]);
#pragma omp parallel for schedule(dynamic, 1)
    for (int q = 0; q < nblk[l]; ++q) {
      Csr<T> B = submatrix(P->Ahat, b[q], b[q + 1], b[q], b[q + 1]);
      add_diag(B, sigma);
      f[q] = factor(B, ilu_type, tau, lfil, errs[q]);
    }
    for (int q = 0; q < nblk[l]; ++q)
      if (!errs[q].empty()) { err = errs[q] + " (level " + std::to_string(l) + ", block " + std::to_string(q) + ")"; delete P; return nullptr; }
    P->fac.push_back(std::move(f));
    if (l == 0) P->C0 = submatrix(P->Ahat, P->o[1], n, P->o[1], n);
    P->E.push_back(submatrix(P->Ahat, P->o[l + 1], n, P->o[l], P->o[l + 1]));
    P->F.push_back(submatrix(P->Ahat, P->o[l], P->o[l + 1], P->o[l + 1], n));
  }
  P->last.assign(last_off, last_off + nlast + 1);
  P->lastfac.resize(nlast);
  std::vector<std::string> errs(nlast);
#pragma omp parallel for schedule(dynamic, 1)
  for (int q = 0; q < nlast; ++q) {
    Csr<T> C = submatrix(P->Ahat, P->last[q], P->last[q + 1], P->last[q], P->last[q + 1]);
    add_diag(C, sigma);
    P->lastfac[q] = factor(C, ilu_type, tau, lfil, errs[q]);
  }
  for (int q = 0; q < nlast; ++q)
    if (!errs[q].empty()) { err = errs[q] + " (C_last block " + std::to_string(q) + ")"; delete P; return nullptr; }
  return P;
}

struct Handle {
  int is_cplx = 0;
  void *p = nullptr;
  std::vector<int64_t> perm;
};

struct IluHandle {
  int is_cplx = 0;
  void *f = nullptr;
};

void set_err(char *err, int cap, const std::string &s) {
  if (err && cap > 0) { std::snprintf(err, (size_t)cap, "%s", s.c_str()); }
}

template <typename T>
void copy_csr(const Csr<T> &A, int64_t *ptr, int64_t *col, void *val) {
  std::copy(A.ptr.begin(), A.ptr.end(), ptr);
  std::copy(A.col.begin(), A.col.end(), col);
  std::copy(A.val.begin(), A.val.end(), static_cast<T *>(val));
}

}  // namespace

// ============================================================================
// extern "C" surface for tests/oracle_py.py (ctypes)
// ============================================================================
extern "C" {

// OpenMP threads of the oracle (results do not depend on it; bench.py times 1 and all cores)
void or_set_threads(int n) {
#ifdef _OPENMP
  omp_set_num_threads(n > 0 ? n : 1);
#else
  (void)n;
#endif
}
int or_get_threads() {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

void or_spmv(int cplx, int64_t n, const int64_t *rowptr, const int32_t *col, const void *val,
             const void *x, void *y) {
  if (cplx) {
    Csr<zc> A = make_csr<zc>(n, rowptr, col, val);
    spmv(A, static_cast<const zc *>(x), static_cast<zc *>(y));
  } else {
    Csr<double> A = make_csr<double>(n, rowptr, col, val);
    spmv(A, static_cast<const double *>(x), static_cast<double *>(y));
  }
}

// ---- standalone ILU on one matrix (for pins and for verifying bundle factors)
void *or_ilu_create(int cplx, int64_t n, const int64_t *rowptr, const int32_t *col, const void *val,
                    int type, double tau, int lfil, char *err, int errcap) {
  std::string e;
  auto *h = new IluHandle();
  h->is_cplx = cplx;
  if (cplx) {
    Csr<zc> A = make_csr<zc>(n, rowptr, col, val);
    auto *f = new Ilu<zc>(factor(A, type, tau, lfil, e));
    h->f = f;
  } else {
    Csr<double> A = make_csr<double>(n, rowptr, col, val);
    auto *f = new Ilu<double>(factor(A, type, tau, lfil, e));
    h->f = f;
  }
  if (!e.empty()) { set_err(err, errcap, e); return nullptr; }
  return h;
}

int64_t or_ilu_nnz(void *hv, int which) {
  auto *h = static_cast<IluHandle *>(hv);
  if (h->is_cplx) { auto *f = static_cast<Ilu<zc> *>(h->f); return which ? f->U.nnz() : f->L.nnz(); }
  auto *f = static_cast<Ilu<double> *>(h->f);
  return which ? f->U.nnz() : f->L.nnz();
}


void or_ilu_get(void *hv, int which, int64_t *ptr, int64_t *col, void *val) {
  auto *h = static_cast<IluHandle *>(hv);
  if (h->is_cplx) { auto *f = static_cast<Ilu<zc> *>(h->f); copy_csr(which ? f->U : f->L, ptr, col, val); }
  else { auto *f = static_cast<Ilu<double> *>(h->f); copy_csr(which ? f->U : f->L, ptr, col, val); }
}

void or_ilu_solve(void *hv, const void *b, void *x) {
  auto *h = static_cast<IluHandle *>(hv);
  if (h->is_cplx) lusolve(*static_cast<Ilu<zc> *>(h->f), static_cast<const zc *>(b), static_cast<zc *>(x));
  else lusolve(*static_cast<Ilu<double> *>(h->f), static_cast<const double *>(b), static_cast<double *>(x));
}

void or_ilu_destroy(void *hv) {
  auto *h = static_cast<IluHandle *>(hv);
  if (!h) return;
  if (h->is_cplx) delete static_cast<Ilu<zc> *>(h->f); else delete static_cast<Ilu<double> *>(h->f);
  delete h;
}

// ---- the preconditioner ----------------------------------------------------
void *or_precond_create(int cplx, int64_t n, const int64_t *rowptr, const int32_t *col, const void *val,
                        const int64_t *perm, int L, const int64_t *level_off,
                        const int32_t *nblk, const int64_t *blk_off, int nlast, const int64_t *last_off,
                        int ilu_type, double tau, int lfil, double shift, char *err, int errcap) {
  std::string e;
  auto *h = new Handle();
  h->is_cplx = cplx;
  h->perm.assign(perm, perm + n);
  if (cplx) h->p = build_precond<zc>(n, rowptr, col, val, perm, L, level_off, nblk, blk_off, nlast, last_off, ilu_type, tau, lfil, shift, e);
  else h->p = build_precond<double>(n, rowptr, col, val, perm, L, level_off, nblk, blk_off, nlast, last_off, ilu_type, tau, lfil, shift, e);
  if (!h->p) { set_err(err, errcap, e); delete h; return nullptr; }
  return h;
}

void or_precond_destroy(void *hv) {
  auto *h = static_cast<Handle *>(hv);
  if (!h) return;
  if (h->is_cplx) delete static_cast<Precond<zc> *>(h->p); else delete static_cast<Precond<double> *>(h->p);
  delete h;
}

void or_precond_set_root_its(void *hv, int its) {
  auto *h = static_cast<Handle *>(hv);
  if (h->is_cplx) static_cast<Precond<zc> *>(h->p)->root_its = its;
  else static_cast<Precond<double> *>(h->p)->root_its = its;
}

void or_precond_set_lowrank(void *hv, int l, int k, const void *W, const void *G) {
  auto *h = static_cast<Handle *>(hv);
  if (h->is_cplx) {
    auto *P = static_cast<Precond<zc> *>(h->p);
    const int64_t sl = P->s(l);
    P->k[l] = k;
    P->W[l].assign(static_cast<const zc *>(W), static_cast<const zc *>(W) + sl * k);
    P->G[l].assign(static_cast<const zc *>(G), static_cast<const zc *>(G) + (int64_t)k * k);
  } else {
    auto *P = static_cast<Precond<double> *>(h->p);
    const int64_t sl = P->s(l);
    P->k[l] = k;
    P->W[l].assign(static_cast<const double *>(W), static_cast<const double *>(W) + sl * k);
    P->G[l].assign(static_cast<const double *>(G), static_cast<const double *>(G) + (int64_t)k * k);
  }
}

// y = M^{-1} r in the permuted order (c4) ; l0 > 0 gives C_{l0-1}^{-1} on [o_{l0}, N)
void or_precond_apply_from(void *hv, int l0, const void *r, void *y) {
  auto *h = static_cast<Handle *>(hv);
  if (h->is_cplx) static_cast<Precond<zc> *>(h->p)->apply_from(l0, static_cast<const zc *>(r), static_cast<zc *>(y));
  else static_cast<Precond<double> *>(h->p)->apply_from(l0, static_cast<const double *>(r), static_cast<double *>(y));
}

void or_ghat(void *hv, int l, const void *v, void *out) {
  auto *h = static_cast<Handle *>(hv);
  if (h->is_cplx) static_cast<Precond<zc> *>(h->p)->ghat(l, static_cast<const zc *>(v), static_cast<zc *>(out));
  else static_cast<Precond<double> *>(h->p)->ghat(l, static_cast<const double *>(v), static_cast<double *>(out));
}

// natural-order preconditioner M_nat^{-1} = P M^{-1} Pᵀ (reading Q21); usable as precond_fn
void or_precond_natural(void *hv, const void *in, void *out) {
  auto *h = static_cast<Handle *>(hv);
  const int64_t n = (int64_t)h->perm.size();
  if (h->is_cplx) {
    const zc *x = static_cast<const zc *>(in);
    std::vector<zc> a(n), b(n);
#pragma omp parallel for schedule(static) if (n > 4096)
    for (int64_t i = 0; i < n; ++i) a[i] = x[h->perm[i]];
    static_cast<Precond<zc> *>(h->p)->apply_from(0, a.data(), b.data());
    zc *y = static_cast<zc *>(out);
#pragma omp parallel for schedule(static) if (n > 4096)
    for (int64_t i = 0; i < n; ++i) y[h->perm[i]] = b[i];
  } else {
    const double *x = static_cast<const double *>(in);
    std::vector<double> a(n), b(n);
#pragma omp parallel for schedule(static) if (n > 4096)
    for (int64_t i = 0; i < n; ++i) a[i] = x[h->perm[i]];
    static_cast<Precond<double> *>(h->p)->apply_from(0, a.data(), b.data());
    double *y = static_cast<double *>(out);
#pragma omp parallel for schedule(static) if (n > 4096)
    for (int64_t i = 0; i < n; ++i) y[h->perm[i]] = b[i];
  }
}

// Factor of level l (l == L: C_last), block q; which = 0 (L) / 1 (U).
int64_t or_precond_factor_nnz(void *hv, int l, int q, int which) {
  auto *h = static_cast<Handle *>(hv);
  if (h->is_cplx) {
    auto *P = static_cast<Precond<zc> *>(h->p);
    const Ilu<zc> &f = (l == P->L) ? P->lastfac[q] : P->fac[l][q];
    return which ? f.U.nnz() : f.L.nnz();
  }
  auto *P = static_cast<Precond<double> *>(h->p);
  const Ilu<double> &f = (l == P->L) ? P->lastfac[q] : P->fac[l][q];
  return which ? f.U.nnz() : f.L.nnz();
}

void or_precond_factor_get(void *hv, int l, int q, int which, int64_t *ptr, int64_t *col, void *val) {
  auto *h = static_cast<Handle *>(hv);
  if (h->is_cplx) {
    auto *P = static_cast<Precond<zc> *>(h->p);
    const Ilu<zc> &f = (l == P->L) ? P->lastfac[q] : P->fac[l][q];
    copy_csr(which ? f.U : f.L, ptr, col, val);
  } else {
    auto *P = static_cast<Precond<double> *>(h->p);
    const Ilu<double> &f = (l == P->L) ? P->lastfac[q] : P->fac[l][q];
    copy_csr(which ? f.U : f.L, ptr, col, val);
  }
}

// FGMRES(m) (c5) on natural-order A with a precond_fn (NULL = identity).
// Returns status (0 converged, 1 not converged); hist receives relative
// residual estimates (entry 0 = initial); diag[0..2] = max_orth, max_arnoldi,
// max_est_gap when want_diag != 0.
int or_fgmres(int cplx, int64_t n, const int64_t *rowptr, const int32_t *col, const void *val,
              precond_fn M, void *Muser, const void *b, void *x, double rtol, int restart, int maxit,
              int *its, double *hist, int histcap, int *histlen, double *final_relres,
              int want_diag, double *diag) {
  auto fill = [&](auto &o) {
    *its = o.its;
    int hl = (int)o.hist.size();
    *histlen = hl;
    for (int i = 0; i < hl && i < histcap; ++i) hist[i] = o.hist[i];
    *final_relres = o.final_relres;
    if (want_diag && diag) { diag[0] = o.max_orth; diag[1] = o.max_arnoldi; diag[2] = o.max_est_gap; }
    return o.status;
  };
  if (cplx) {
    Csr<zc> A = make_csr<zc>(n, rowptr, col, val);
    auto o = fgmres(A, M, Muser, static_cast<const zc *>(b), static_cast<zc *>(x), rtol, restart, maxit, want_diag != 0);
    return fill(o);
  }
  Csr<double> A = make_csr<double>(n, rowptr, col, val);
  auto o = fgmres(A, M, Muser, static_cast<const double *>(b), static_cast<double *>(x), rtol, restart, maxit, want_diag != 0);
  return fill(o);
}

// The same with DCGS2 (c5', reading Q38).
int or_fgmres_dcgs2(int cplx, int64_t n, const int64_t *rowptr, const int32_t *col, const void *val,
                    precond_fn M, void *Muser, const void *b, void *x, double rtol, int restart, int maxit,
                    int *its, double *hist, int histcap, int *histlen, double *final_relres,
                    int want_diag, double *diag) {
  auto fill = [&](auto &o) {
    *its = o.its;
    int hl = (int)o.hist.size();
    *histlen = hl;
    for (int i = 0; i < hl && i < histcap; ++i) hist[i] = o.hist[i];
    *final_relres = o.final_relres;
    if (want_diag && diag) { diag[0] = o.max_orth; diag[1] = o.max_arnoldi; diag[2] = o.max_est_gap; }
    return o.status;
  };
  if (cplx) {
    Csr<zc> A = make_csr<zc>(n, rowptr, col, val);
    auto o = fgmres_dcgs2(A, M, Muser, static_cast<const zc *>(b), static_cast<zc *>(x), rtol, restart, maxit,
                          want_diag != 0);
    return fill(o);
  }
  Csr<double> A = make_csr<double>(n, rowptr, col, val);
  auto o = fgmres_dcgs2(A, M, Muser, static_cast<const double *>(b), static_cast<double *>(x), rtol, restart, maxit,
                        want_diag != 0);
  return fill(o);
}

}  // extern "C"
