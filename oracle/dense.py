"""ORACLE — test infrastructure only.  Plain NumPy/SciPy dense helpers.

* tiny_structure: a simple multilevel p-way vertex-separator structure for
  tiny grids (recursive coordinate bisection, Alg. 3
  P:L582-597).  It exists so the oracle can be pinned on its own (exact-mode
  checks) without the product's setup.  Any valid structure serves.
* dense_lowrank: the rank-k term of eq. (gemslr6)/(gemslr5) (P:L417-427,
  P:L509-511) from a DENSE Schur decomposition of Ĝ_l, with the
  Schur vectors sorted by |γ/(1-γ)| descending (reading Q6).
* verify_*: the independent bundle checks of SURVEY.md §8(c) c3.
"""
from __future__ import annotations

import numpy as np
import scipy.linalg as sla
import scipy.sparse as sp


# ---------------------------------------------------------------------------
# tiny structure (oracle-only)
# ---------------------------------------------------------------------------
def _sym_graph(A):
    P = abs(A) + abs(A.T)
    P = sp.csr_matrix(P)
    P.setdiag(0)
    P.eliminate_zeros()
    return P


def _bisect_parts(verts, coords, p):
    """Recursive coordinate bisection of `verts` into p parts (lists)."""
    if p == 1:
        return [verts]
    pa = p // 2
    c = coords[verts]
    ext = c.max(axis=0) - c.min(axis=0)
    ax = int(np.argmax(ext))
    order = verts[np.lexsort((verts, c[:, ax]))]
    na = len(verts) * pa // p
    return _bisect_parts(np.sort(order[:na]), coords, pa) + _bisect_parts(np.sort(order[na:]), coords, p - pa)


def tiny_structure(A, coords, levels, p, nlast=None):
    """Multilevel p-way vertex separators by coordinate bisection.

    Level l partitions the induced subgraph on the previous separator into p
    parts; a vertex joins the separator when it has a neighbour in a part of
    higher id (a vertex cover of the cut edges), so no edge joins two parts
    (P:L576-579).  Stops early when the separator has < 2p vertices.
    Returns the structure dict consumed by oracle.Precond.
    """
    A = sp.csr_matrix(A)
    G = _sym_graph(A)
    n = A.shape[0]
    current = np.arange(n)
    perm_parts, level_off, blocks = [], [0], []
    pos = 0
    for l in range(levels):
        if len(current) < 2 * p and l > 0:
            break
        parts = _bisect_parts(current, coords, p)
        part_of = -np.ones(n, dtype=np.int64)
        for q, vs in enumerate(parts):
            part_of[vs] = q
        sep = []
        for v in current:
            nb = G.indices[G.indptr[v]:G.indptr[v + 1]]
            nb = nb[part_of[nb] >= 0]
            if np.any(part_of[nb] > part_of[v]):
                sep.append(v)
        sep = np.array(sorted(sep), dtype=np.int64)
        insep = np.zeros(n, dtype=bool)
        insep[sep] = True
        bl = [pos]
        for vs in parts:
            inner = np.array([v for v in vs if not insep[v]], dtype=np.int64)
            perm_parts.append(inner)
            pos += len(inner)
            bl.append(pos)
        blocks.append(np.array(bl, dtype=np.int64))
        level_off.append(pos)
        current = sep
    perm_parts.append(current)
    perm = np.concatenate(perm_parts).astype(np.int64)
    s = len(current)
    nlast = nlast or p
    nlast = max(1, min(nlast, s))
    last = level_off[-1] + np.array([s * q // nlast for q in range(nlast + 1)], dtype=np.int64)
    return dict(perm=perm, level_off=np.array(level_off, dtype=np.int64), blocks=blocks, last_off=last)


# ---------------------------------------------------------------------------
# dense low rank (oracle-only)
# ---------------------------------------------------------------------------
def dense_ghat(P, l):
    """Ĝ_l as a dense s_l x s_l matrix, column by column through the oracle."""
    s = P.s(l)
    Gm = np.zeros((s, s), dtype=P.dtype)
    e = np.zeros(s, dtype=P.dtype)
    for j in range(s):
        e[:] = 0
        e[j] = 1
        Gm[:, j] = P.ghat(l, e)
    return Gm


def lowrank_from_dense(Gm, k=None, real=None):
    """(W, R, G) with G = (I-R)^{-1} - I from a dense Schur decomposition of Ĝ.

    k=None: full rank with W = I, R = Ĝ (the correction W[(I-R)^{-1}-I]W^H is
    basis-invariant).  Otherwise the k leading Schur vectors by
    |γ/(1-γ)|; real Ĝ keeps a real quasi-triangular Schur form
    and never splits a conjugate pair (reading Q7).
    """
    s = Gm.shape[0]
    if real is None:
        real = not np.iscomplexobj(Gm)
    if k is None or k >= s:
        W = np.eye(s, dtype=Gm.dtype)
        R = Gm.copy()
    else:
        ev = np.linalg.eigvals(Gm)
        key = np.abs(ev / (1.0 - ev))
        thr = np.sort(key)[::-1][k - 1]
        tol = 1e-12 * max(1.0, thr)
        def wanted(z):
            return abs(z / (1.0 - z)) >= thr - tol
        if real:
            T, Z, sdim = sla.schur(Gm, output="real", sort=lambda re, im: wanted(complex(re, im)))
        else:
            T, Z, sdim = sla.schur(Gm, output="complex", sort=wanted)
        W = Z[:, :sdim]
        R = T[:sdim, :sdim]
    I = np.eye(R.shape[0], dtype=R.dtype)
    G = np.linalg.inv(I - R) - I
    return W, R, G


def smw_inverse(Cm, W, R):
    """S^{-1} = C^{-1} + C^{-1} W [(I-R)^{-1} - I] W^H  (eq. gemslr4)."""
    Ci = np.linalg.inv(Cm)
    I = np.eye(R.shape[0], dtype=R.dtype)
    return Ci + Ci @ W @ (np.linalg.inv(I - R) - I) @ W.conj().T


# ---------------------------------------------------------------------------
# bundle verification — all computed from the oracle's own Â
# ---------------------------------------------------------------------------
def permute_matrix(A, perm):
    """Â = Pᵀ A P with perm[new] = old."""
    A = sp.csr_matrix(A)
    return A[perm][:, perm].tocsr()


def verify_perm(perm, n):
    perm = np.asarray(perm)
    return len(perm) == n and np.array_equal(np.sort(perm), np.arange(n))


def verify_separators(Ahat, level_off, blocks):
    """No nonzero of Â couples two different blocks inside I_l, for every level."""
    Ahat = sp.coo_matrix(Ahat)
    bad = 0
    for l, bl in enumerate(blocks):
        o0, o1 = level_off[l], level_off[l + 1]
        m = (Ahat.row >= o0) & (Ahat.row < o1) & (Ahat.col >= o0) & (Ahat.col < o1)
        r, c = Ahat.row[m], Ahat.col[m]
        br = np.searchsorted(bl, r, side="right")
        bc = np.searchsorted(bl, c, side="right")
        bad += int(np.count_nonzero(br != bc))
    return bad


def ilu0_property_error(B, Lf, Uf):
    """max |(LU)_ij - b_ij| / max|b| over pattern(B), with L unit lower (strict part given)."""
    B = sp.csr_matrix(B)
    n = B.shape[0]
    Lfull = sp.csr_matrix(Lf) + sp.identity(n, dtype=B.dtype, format="csr")
    LU = (Lfull @ sp.csr_matrix(Uf)).tocsr()
    Bc = B.tocoo()
    vals = np.asarray(LU[Bc.row, Bc.col]).ravel()
    return float(np.max(np.abs(vals - Bc.data)) / np.max(np.abs(Bc.data)))


def pattern_equal(A, Bm):
    A = sp.csr_matrix(A)
    Bm = sp.csr_matrix(Bm)
    A.sort_indices()
    Bm.sort_indices()
    return np.array_equal(A.indptr, Bm.indptr) and np.array_equal(A.indices, Bm.indices)


# ---------------------------------------------------------------------------
# vectorised setup for the bench reference arm (oracle-only; timing, not parity)
# ---------------------------------------------------------------------------
def rcb_structure(A, coords, levels, p, nlast=None):
    """Multilevel p-way vertex separators (Alg. 3) by recursive
    coordinate bisection, vectorised for large grids.  Same rules as
    tiny_structure: a vertex joins the separator when it has a neighbour of
    higher part id; stop when the separator has < 2p vertices."""
    A = sp.csr_matrix(A)
    G = _sym_graph(A).tocoo()
    n = A.shape[0]
    current = np.arange(n)
    perm_parts, level_off, blocks = [], [0], []
    pos = 0

    def bisect(verts, q, first, part):
        if q == 1:
            part[verts] = first
            return
        qa = q // 2
        c = coords[verts]
        ax = int(np.argmax(c.max(axis=0) - c.min(axis=0)))
        order = verts[np.lexsort((verts, c[:, ax]))]
        na = len(verts) * qa // q
        bisect(np.sort(order[:na]), qa, first, part)
        bisect(np.sort(order[na:]), q - qa, first + qa, part)

    for l in range(levels):
        if len(current) < 2 * p and l > 0:
            break
        part = -np.ones(n, dtype=np.int64)
        bisect(current, p, 0, part)
        u, v = G.row, G.col
        m = (part[u] >= 0) & (part[v] >= 0) & (part[v] > part[u])
        insep = np.zeros(n, dtype=bool)
        insep[u[m]] = True
        sep = current[insep[current]]
        bl = [pos]
        inner_all = current[~insep[current]]
        pa = part[inner_all]
        order = np.lexsort((inner_all, pa))
        inner_sorted = inner_all[order]
        counts = np.bincount(pa, minlength=p)
        perm_parts.append(inner_sorted)
        for q in range(p):
            pos += int(counts[q])
            bl.append(pos)
        blocks.append(np.array(bl, dtype=np.int64))
        level_off.append(pos)
        current = np.sort(sep)
    perm_parts.append(current)
    perm = np.concatenate(perm_parts).astype(np.int64)
    s = len(current)
    nlast = nlast or p
    nlast = max(1, min(nlast, s))
    last = level_off[-1] + np.array([s * q // nlast for q in range(nlast + 1)], dtype=np.int64)
    return dict(perm=perm, level_off=np.array(level_off, dtype=np.int64), blocks=blocks, last_off=last)


def arnoldi_lowrank(P, k, seed=0):
    """Rank-k terms bottom-up from ONE Arnoldi cycle of length
    m = 2k on Ĝ_l with CGS2, Schur of H_m sorted by
    |γ/(1-γ)| (real Schur for real problems, pairs kept).  Installs W_l, G_l
    into the oracle preconditioner.  (Reference-arm setup: no thick restart.)"""
    if k <= 0:
        return
    rng = np.random.default_rng(seed)
    L = len(P.o) - 1
    for l in range(L - 1, -1, -1):
        s = P.s(l)
        if s == 0:
            continue
        m = min(2 * k, s)
        V = np.zeros((s, m + 1), dtype=P.dtype)
        H = np.zeros((m + 1, m), dtype=P.dtype)
        v0 = rng.uniform(-1, 1, s).astype(P.dtype)
        V[:, 0] = v0 / np.linalg.norm(v0)
        mm = m
        for j in range(m):
            w = P.ghat(l, V[:, j])
            h = V[:, :j + 1].conj().T @ w
            w = w - V[:, :j + 1] @ h
            h2 = V[:, :j + 1].conj().T @ w
            w = w - V[:, :j + 1] @ h2
            H[:j + 1, j] = h + h2
            H[j + 1, j] = np.linalg.norm(w)
            if H[j + 1, j] <= 1e-14 * np.linalg.norm(h):
                mm = j + 1
                break
            V[:, j + 1] = w / H[j + 1, j]
        W, R, G = lowrank_from_dense(H[:mm, :mm], k=min(k, mm))
        P.set_lowrank(l, V[:, :mm] @ W, G)
