// Host stage of setup(A, levels, p, rank): Alg. 1 pGeMSLRSetup lines 1-5
// except the low-rank terms.  Validate A, reorder (Alg. 3), form
// Â = Pᵀ A P, cut it into B_l blocks / E_l / F_l / C_last blocks
// (P:L458-464), factor every block in parallel and
// build the level-scheduled sweeps.
#include <chrono>
#include <cstdio>
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <type_traits>

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

// Complex diagonal shift during the block ILUs ("a complex shift
// equal to 0.05 i Σ_i |A_ii| / n_A during the ILU factorization of the
// on-diagonal blocks"): sigma = i * opt.shift * Σ|a_ii| / n, added to the
// diagonal of every B_l block and every C_last block before factoring (Q33).
template <typename T> T ilu_sigma(const Csr<T> &, double) { return T(0); }
template <> zc ilu_sigma<zc>(const Csr<zc> &A, double factor) {
  if (factor == 0.0) return zc(0);
  double s = 0;
  for (int64_t i = 0; i < A.n; ++i)
    for (int64_t p = A.ptr[i]; p < A.ptr[i + 1]; ++p)
      if (A.col[p] == i) s += std::abs(A.val[p]);
  return zc(0.0, factor * s / (double)A.n);
}
template <typename T>
void shift_diag(Csr<T> &B, T sigma) {
  if (sigma == T(0)) return;
  for (int64_t i = 0; i < B.n; ++i)
    for (int64_t p = B.ptr[i]; p < B.ptr[i + 1]; ++p)
      if (B.col[p] == i) B.val[p] += sigma;
}

template <typename T>
bool factor_blocks(const Csr<T> &Ahat, const std::vector<int64_t> &bl, const SetupOptions &opt, T sigma,
                   std::vector<Factor<T>> &out, const std::string &where, Error &err) {
  const int nb = (int)bl.size() - 1;
  out.assign(nb, Factor<T>());
  std::vector<std::string> errs(nb);
  std::vector<char> ok(nb, 1);
#pragma omp parallel for schedule(dynamic, 1)
  for (int q = 0; q < nb; ++q) {
    Csr<T> B = sub(Ahat, bl[q], bl[q + 1], bl[q], bl[q + 1], true);
    shift_diag(B, sigma);
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
// Clusters per block of a stage's triangular solves (plan.hpp, split form): the
// subdomains of level 0 are few (p / nranks) and deep, so each is cut into Q
// chunks on Q SMs; stages with small blocks keep one CTA per block.
static int split_for(const std::vector<int64_t> &bl, const SetupOptions &opt, bool is_complex) {
  if (opt.split == 1) return 1;
  int nb = 0;
  int64_t rows = 0;
  for (size_t q = 0; q + 1 < bl.size(); ++q)
    if (bl[q + 1] > bl[q]) { nb++; rows += bl[q + 1] - bl[q]; }
  if (nb == 0) return 1;
  if (opt.split >= 2) return opt.split;
  // complex (C4, 64 blocks: Q = 2): measured 278 / 290 us per level-0 sweep pair vs
  // 268 / 284 unsplit (15 warps either way) — the split only pays in fp64
  if (is_complex) return 1;
  const int64_t avg = rows / nb;
  // Measured (tools/split_cmp.py, level-0 DOWN / UP per apply): C5 (32 blocks of 60k rows,
  // ~6 slices per level) Q = 4 228 / 236 us vs 281 / 299 unsplit (Q = 2: 267 / 282); C3 (64
  // blocks of 30k rows, only Q = 2 fits) 194 / 198 vs 181 / 186; C2 (16 blocks of 15k rows)
  // Q = 4 111 / 111, Q = 2 105 / 105 vs 98 / 99.  The split pays only for blocks whose levels
  // carry many slices: Q = 4 with chunks of at least 12k rows (blocks >= 48k rows).
  // (Experiments: GEMSLR_SPLIT_MAX, GEMSLR_SPLIT_MINROWS.)
  static const int qmax = getenv("GEMSLR_SPLIT_MAX") ? atoi(getenv("GEMSLR_SPLIT_MAX")) : 4;
  static const int64_t minrows = getenv("GEMSLR_SPLIT_MINROWS") ? atoll(getenv("GEMSLR_SPLIT_MINROWS")) : 12288;
  const int qmin = getenv("GEMSLR_SPLIT_MAX") ? 2 : 4;
  for (int Q = 4; Q >= qmin; Q /= 2) {
    if (Q > qmax) continue;
    const int fit = Q == 4 ? opt.sms - 16 : opt.sms;                // clusters of 4 leave a few SMs of each GPC idle
    if ((int64_t)nb * Q <= fit && avg / Q >= minrows) return Q;
  }
  return 1;
}

template <typename T>
void make_stage(const std::vector<int64_t> &bl, const std::vector<Factor<T>> &fac, Stage<T> &S, int Q = 1,
                const std::vector<int64_t> *tails = nullptr) {
  std::vector<int64_t> bounds, tl;
  std::vector<Factor<T>> facs;
  for (size_t q = 0; q + 1 < bl.size(); ++q) {
    if (bl[q + 1] == bl[q]) continue;
    if (bounds.empty() || bounds.back() != bl[q]) bounds.push_back(bl[q]);
    bounds.push_back(bl[q + 1]);
    facs.push_back(fac[q]);
    if (tails) tl.push_back((*tails)[q]);
  }
  if (bounds.empty()) bounds.push_back(bl.empty() ? 0 : bl[0]);
  pack_stage(bounds, facs, S, Q, tails && !facs.empty() ? &tl : nullptr);
}

}  // namespace

// Halo plan of this rank from every rank's sorted list of needed remote
// positions (all ranks compute the same lists, so sends and receives match).
static HaloPlan make_halo(int rank, int nranks, const std::vector<int32_t> &owner, const std::vector<int64_t> &loc,
                          const std::vector<std::vector<int64_t>> &needed) {
  HaloPlan h;
  std::vector<std::vector<int64_t>> sendto(nranks), recvfrom(nranks);
  for (int64_t pos : needed[rank]) recvfrom[owner[pos]].push_back(pos);
  for (int r = 0; r < nranks; ++r) {
    if (r == rank) continue;
    for (int64_t pos : needed[r])
      if (owner[pos] == rank) sendto[r].push_back(pos);
  }
  for (int r = 0; r < nranks; ++r) {
    if (r == rank || (sendto[r].empty() && recvfrom[r].empty())) continue;
    h.peer.push_back(r);
    for (int64_t pos : sendto[r]) { h.sidx.push_back((int32_t)loc[pos]); h.sglob.push_back(pos); }
    for (int64_t pos : recvfrom[r]) h.rglob.push_back(pos);
    h.soff.push_back((int64_t)h.sidx.size());
    h.roff.push_back((int64_t)h.rglob.size());
  }
  return h;
}

// needed[r]: sorted unique remote positions referenced by rank r's rows
// [r0, r1) of M (columns in [c0, c1), excluding `skip_from` and above).
template <typename T>
static std::vector<std::vector<int64_t>> needed_sets(const Csr<T> &M, int nranks, const std::vector<int32_t> &owner,
                                                     int64_t r0, int64_t r1, int64_t c0, int64_t c1) {
  std::vector<std::vector<int64_t>> need(nranks);
  for (int64_t i = r0; i < r1; ++i) {
    const int r = owner[i];
    for (int64_t p = M.ptr[i]; p < M.ptr[i + 1]; ++p) {
      const int64_t j = M.col[p];
      if (j >= c0 && j < c1 && owner[j] != r) need[r].push_back(j);
    }
  }
  for (auto &v : need) {
    std::sort(v.begin(), v.end());
    v.erase(std::unique(v.begin(), v.end()), v.end());
  }
  return need;
}

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
  const int G = opt.nranks, me = opt.rank;
  if (G < 1 || me < 0 || me >= G || opt.p % G != 0) {
    err = {-1, "INVALID_ARG: subdomains must be a multiple of the number of ranks (P:L76)"};
    return false;
  }
  Graph g = build_graph(n, rowptr, colidx);
  const auto tq0 = std::chrono::steady_clock::now();
  auto tdbg = [&](const char *what) {
    if (getenv("GEMSLR_DEBUG_TAIL"))
      fprintf(stderr, "setup %s %.2f s\n", what, std::chrono::duration<double>(std::chrono::steady_clock::now() - tq0).count());
  };
  if (!build_structure(g, opt, plan.st, err)) return false;
  tdbg("structure");
  const Structure &st = plan.st;
  plan.Ahat = permute(n, rowptr, colidx, vals, st);
  const Csr<T> &Ah = plan.Ahat;
  const T sigma = ilu_sigma<T>(Ah, opt.shift);                     // Σ|a_ii| is invariant under the permutation
  const int L = st.L;
  plan.nranks = G;
  plan.rank = me;
  // ---- ownership: level-0 parts in contiguous rank ranges;
  // a part of a later level (and a C_last row) goes to the rank owning most of
  // its neighbours in earlier levels (ties -> lower rank)
  std::vector<int32_t> &owner = plan.owner;
  owner.assign(n, 0);
  std::vector<std::vector<int32_t>> blk_owner(L);
  auto vote = [&](int64_t r0, int64_t r1, int64_t below) {
    std::vector<int64_t> v(G, 0);
    for (int64_t i = r0; i < r1; ++i)
      for (int64_t p = Ah.ptr[i]; p < Ah.ptr[i + 1]; ++p)
        if (Ah.col[p] < below) v[owner[Ah.col[p]]]++;
    int best = 0;
    for (int r = 1; r < G; ++r)
      if (v[r] > v[best]) best = r;
    return best;
  };
  for (int l = 0; l < L; ++l) {
    const auto &bl = st.blk[l];
    const int nb = (int)bl.size() - 1;
    blk_owner[l].assign(nb, 0);
    for (int q = 0; q < nb; ++q) {
      const int r = (l == 0) ? (int)((int64_t)q * G / nb) : (G == 1 ? 0 : vote(bl[q], bl[q + 1], st.o[l]));
      blk_owner[l][q] = r;
      for (int64_t i = bl[q]; i < bl[q + 1]; ++i) owner[i] = r;
    }
  }
  if (G > 1)
    for (int64_t i = st.o[L]; i < n; ++i) owner[i] = vote(i, i + 1, st.o[L]);
  // ---- local layout
  std::vector<int64_t> loc(n, -1);
  plan.gpos.clear();
  plan.lo.assign(L + 1, 0);
  for (int l = 0; l <= L; ++l) {
    plan.lo[l] = (int64_t)plan.gpos.size();
    const int64_t a = st.o[l], b = (l == L) ? n : st.o[l + 1];
    for (int64_t i = a; i < b; ++i)
      if (owner[i] == me) { loc[i] = (int64_t)plan.gpos.size(); plan.gpos.push_back(i); }
  }
  plan.nloc = (int64_t)plan.gpos.size();
  plan.slast = n - st.o[L];
  const int64_t nloc = plan.nloc;
  plan.last_idx.clear();
  for (int64_t j = plan.lo[L]; j < nloc; ++j) plan.last_idx.push_back((int32_t)(plan.gpos[j] - st.o[L]));
  // ---- halo plans
  plan.hA = make_halo(me, G, owner, loc, needed_sets(Ah, G, owner, 0, n, 0, n));
  plan.hE.assign(L, HaloPlan());
  plan.hF.assign(L, HaloPlan());
  for (int l = 0; l < L; ++l) {
    plan.hE[l] = make_halo(me, G, owner, loc, needed_sets(Ah, G, owner, st.o[l + 1], n, st.o[l], st.o[l + 1]));
    const int64_t fcend = (G > 1) ? st.o[L] : n;       // C_last is replicated when G > 1
    plan.hF[l] = make_halo(me, G, owner, loc, needed_sets(Ah, G, owner, st.o[l], st.o[l + 1], st.o[l + 1], fcend));
  }
  auto halo_index = [](const HaloPlan &h) {
    std::vector<std::pair<int64_t, int64_t>> m;
    for (int64_t i = 0; i < (int64_t)h.rglob.size(); ++i) m.push_back({h.rglob[i], i});
    std::sort(m.begin(), m.end());
    return m;
  };
  auto lookup = [](const std::vector<std::pair<int64_t, int64_t>> &m, int64_t pos) {
    auto it = std::lower_bound(m.begin(), m.end(), std::make_pair(pos, (int64_t)-1));
    return it->second;
  };
  // ---- local operators with remapped columns
  auto local_rows = [&](int64_t lr0, int64_t lr1, int64_t c0, int64_t c1, const HaloPlan &h, bool clast_rep) {
    Csr<T> M;
    M.n = lr1 - lr0;
    M.ptr.assign(M.n + 1, 0);
    const auto idx = halo_index(h);
    const int64_t nh = h.nrecv();
    for (int64_t li = lr0; li < lr1; ++li) {
      const int64_t i = plan.gpos[li];
      for (int64_t p = Ah.ptr[i]; p < Ah.ptr[i + 1]; ++p) {
        const int64_t j = Ah.col[p];
        if (j < c0 || j >= c1) continue;
        int64_t c;
        if (clast_rep && j >= st.o[L]) c = nloc + nh + (j - st.o[L]);
        else if (owner[j] == me) c = loc[j];
        else c = nloc + lookup(idx, j);
        M.col.push_back((int32_t)c);
        M.val.push_back(Ah.val[p]);
      }
      M.ptr[li - lr0 + 1] = (int64_t)M.col.size();
    }
    return M;
  };
  plan.Aloc = local_rows(0, nloc, 0, n, plan.hA, false);
  plan.E.assign(L, Csr<T>());
  plan.F.assign(L, Csr<T>());
  plan.fac.assign(L, {});
  plan.stage.assign(L, Stage<T>());
  plan.fac_nnz = 0;
  for (int l = 0; l < L; ++l) {
    const auto &bl = st.blk[l];
    const int nb = (int)bl.size() - 1;
    // factor the owned blocks only (independent per subdomain)
    std::vector<int64_t> own_bl{bl[0]};
    std::vector<int> own_q;
    for (int q = 0; q < nb; ++q)
      if (blk_owner[l][q] == me) own_q.push_back(q);
    std::vector<Factor<T>> own_fac;
    {
      std::vector<int64_t> b2;
      std::vector<Factor<T>> f2;
      for (int q : own_q) { b2.push_back(bl[q]); b2.push_back(bl[q + 1]); }
      // factor each owned block independently
      const int no = (int)own_q.size();
      f2.assign(no, Factor<T>());
      std::vector<std::string> errs(no);
      std::vector<char> ok(no, 1);
#pragma omp parallel for schedule(dynamic, 1)
      for (int t = 0; t < no; ++t) {
        const int q = own_q[t];
        Csr<T> B = sub(Ah, bl[q], bl[q + 1], bl[q], bl[q + 1], true);
        shift_diag(B, sigma);
        ok[t] = opt.ilu == 0 ? ilu0(B, f2[t], errs[t]) : ilut(B, opt.tau, opt.lfil, f2[t], errs[t]);
      }
      for (int t = 0; t < no; ++t)
        if (!ok[t]) {
          err = {-4, "ZERO_PIVOT: level " + std::to_string(l) + ", block " + std::to_string(own_q[t]) + ": " + errs[t]};
          return false;
        }
      plan.fac[l].assign(nb, Factor<T>());
      for (int t = 0; t < no; ++t) {
        plan.fac_nnz += f2[t].L.nnz() + f2[t].U.nnz();
        plan.fac[l][own_q[t]] = f2[t];
      }
      own_fac = f2;
    }
    // local stage: owned blocks are contiguous in the local layout
    std::vector<int64_t> lb{plan.lo[l]};
    for (size_t t = 0; t < own_q.size(); ++t) lb.push_back(lb.back() + (bl[own_q[t] + 1] - bl[own_q[t]]));
    // tail form (plan.hpp TailPack): a block's tail starts at its first row coupled to a
    // later level (a column of E_l or a row of F_l); every row after it is in the tail
    std::vector<int64_t> tails;
    if (opt.tail) {
      const int64_t a = st.o[l], e = st.o[l + 1];
      std::vector<char> mark(e - a, 0);
      for (int64_t i = a; i < e; ++i)                              // F_l: row i has a later column
        for (int64_t p = Ah.ptr[i]; p < Ah.ptr[i + 1]; ++p)
          if (Ah.col[p] >= e) { mark[i - a] = 1; break; }
      for (int64_t j = e; j < n; ++j)                              // E_l: a later row has column i
        for (int64_t p = Ah.ptr[j]; p < Ah.ptr[j + 1]; ++p)
          if (Ah.col[p] >= a && Ah.col[p] < e) mark[Ah.col[p] - a] = 1;
      for (size_t t = 0; t < own_q.size(); ++t) {
        const int q = own_q[t];
        int64_t f = bl[q + 1];
        for (int64_t i = bl[q]; i < bl[q + 1]; ++i)
          if (mark[i - a]) { f = i; break; }
        tails.push_back(lb[t] + (f - bl[q]));
      }
    }
    tdbg("factors");
    make_stage(lb, own_fac, plan.stage[l], split_for(lb, opt, !std::is_same<T, double>::value),
               opt.tail ? &tails : nullptr);
    plan.E[l] = local_rows(plan.lo[l + 1], nloc, st.o[l], st.o[l + 1], plan.hE[l], false);
    plan.F[l] = local_rows(plan.lo[l], plan.lo[l + 1], st.o[l + 1], n, plan.hF[l], G > 1);
  }
  // C_last: every rank factors and solves all blocks (replicated)
  tdbg("stages");
  if (!factor_blocks(Ah, st.last, opt, sigma, plan.lastfac, "C_last", err)) return false;
  for (auto &f : plan.lastfac) plan.fac_nnz += f.L.nnz() + f.U.nnz();
  std::vector<int64_t> rel;
  for (int64_t v : st.last) rel.push_back(v - st.o[L]);
  make_stage(rel, plan.lastfac, plan.last_stage);
  return true;
}

template bool build_host_plan<double>(int64_t, const int64_t *, const int32_t *, const double *,
                                      const SetupOptions &, HostPlan<double> &, Error &);
template bool build_host_plan<zc>(int64_t, const int64_t *, const int32_t *, const zc *,
                                  const SetupOptions &, HostPlan<zc> &, Error &);

}  // namespace gemslr
