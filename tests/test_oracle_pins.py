"""Pins of the oracle against what the paper and the mathematics fix (CPU only).

Each test names the pin it implements.  A
plausible mistake anywhere in the oracle (a dropped term, a wrong sign or
index, a transposed operand, a missing conjugate) fails at least one:

* SpMV        closed forms (Laplacian·1 = Dirichlet faces), dense product
* ILU(0)      defining property (LU)_ij = b_ij on the pattern; D8 tridiagonal = exact LU
* ILUT        τ=0, lfil=∞ is exact LU (dense solve); identity; lfil cap; monotone accuracy
* apply (c4)  D2 exact mode = Â^{-1} (l_ev 1 and 2, real and complex); D2 ILU(0) +
              full rank = Ŝ^{-1} on the interface; D5 k=0 = dense block-LDU with
              block-Jacobi C; D6 linearity; Ĝ_l against its dense definition
* low rank    D3 SMW identity; D4 eigen-map γ/(1-γ)
* FGMRES (c5) D7 A=I and M=A^{-1} converge in 1 iteration; D1 dense direct solve;
              orthonormality and Arnoldi relation to 1e-12; estimate vs explicit residual
"""
import numpy as np
import pytest
import scipy.linalg as sla
import scipy.sparse as sp

import oracle
from oracle import dense as D
from synth import problems as P


def rng(seed=1):
    return np.random.default_rng(seed)


# ---------------------------------------------------------------- SpMV
def test_spmv_identity_and_2x2():
    I = sp.identity(5, format="csr")
    x = rng().uniform(-1, 1, 5)
    assert np.array_equal(oracle.spmv(I, x), x)
    A = sp.csr_matrix(np.array([[2.0, -1.0], [3.0, 4.0]]))
    assert np.array_equal(oracle.spmv(A, np.array([1.0, 2.0])), np.array([0.0, 11.0]))


def test_spmv_laplacian_ones_is_face_count():
    prob = P.laplacian((5, 4, 3))
    y = oracle.spmv(prob, np.ones(prob.n))
    dims = prob.dims
    crd = prob.coords.astype(int)
    faces = sum((crd[:, a] == 0).astype(int) + (crd[:, a] == d - 1) for a, d in enumerate(dims))
    assert np.array_equal(y, faces.astype(float))


@pytest.mark.parametrize("cplx", [False, True])
def test_spmv_matches_dense_product(cplx):
    r = rng(2)
    M = sp.random(40, 40, density=0.2, random_state=3, format="csr")
    if cplx:
        M = M + 1j * sp.random(40, 40, density=0.2, random_state=4, format="csr")
    M = sp.csr_matrix(M)
    M.sort_indices()
    x = r.uniform(-1, 1, 40) + (1j * r.uniform(-1, 1, 40) if cplx else 0)
    assert np.allclose(oracle.spmv(M, x), M.toarray() @ x, rtol=0, atol=1e-13)


# ---------------------------------------------------------------- ILU
@pytest.mark.parametrize("make", [lambda: P.laplacian((9, 7)), lambda: P.convdiff_upwind((5, 4, 6)),
                                  lambda: P.helmholtz_shifted((4, 5, 3))])
def test_ilu0_defining_property(make):
    prob = make()
    A = prob.scipy()
    f = oracle.Ilu(A, oracle.ILU0)
    assert D.ilu0_property_error(A, f.L, f.U) < 1e-13
    # pattern(L+U) = pattern(A)
    LU = (f.L + f.U).tocsr()
    assert D.pattern_equal(LU, A)


def test_ilu0_tridiagonal_is_exact_lu_D8():
    n = 50
    r = rng(5)
    main = 4 + r.uniform(0, 1, n)
    off1 = r.uniform(-1, 1, n - 1)
    off2 = r.uniform(-1, 1, n - 1)
    A = sp.diags([off2, main, off1], [-1, 0, 1], format="csr")
    b = r.uniform(-1, 1, n)
    x = oracle.Ilu(A, oracle.ILU0).solve(b)
    assert np.allclose(x, np.linalg.solve(A.toarray(), b), rtol=0, atol=1e-12)


@pytest.mark.parametrize("cplx", [False, True])
def test_ilut_exact_when_no_dropping(cplx):
    prob = P.helmholtz_shifted((4, 4, 3)) if cplx else P.convdiff_upwind((4, 5, 3))
    A = prob.scipy()
    f = oracle.Ilu(A, oracle.ILUT, tau=0.0, lfil=10**6)
    n = A.shape[0]
    LU = (f.L + sp.identity(n)) @ f.U
    assert np.abs(LU.toarray() - A.toarray()).max() < 1e-12
    b = rng(6).uniform(-1, 1, n)
    assert np.allclose(f.solve(b), np.linalg.solve(A.toarray(), b), rtol=0, atol=1e-12)


def test_ilut_identity_and_lfil_cap_and_monotone():
    I = sp.identity(7, format="csr")
    f = oracle.Ilu(I, oracle.ILUT, tau=1e-3, lfil=3)
    assert f.L.nnz == 0 and np.array_equal(f.U.toarray(), np.eye(7))
    A = P.laplacian((6, 6, 6)).scipy()
    f = oracle.Ilu(A, oracle.ILUT, tau=1e-4, lfil=3)
    assert np.diff(f.L.indptr).max() <= 3 and np.diff(f.U.indptr).max() <= 4   # + diagonal
    errs = []
    for tau in (1e-1, 1e-2, 0.0):
        g = oracle.Ilu(A, oracle.ILUT, tau=tau, lfil=10**6)
        errs.append(sp.linalg.norm((g.L + sp.identity(A.shape[0])) @ g.U - A))
    assert errs[0] >= errs[1] >= errs[2] and errs[2] < 1e-12


def test_ilut_drops_relative_to_row_norm():
    # 2x2 with a tiny coupling: |a_21/a_11| < τ·||row 2|| -> L entry dropped
    A = sp.csr_matrix(np.array([[1.0, 0.0], [1e-6, 1.0]]))
    f = oracle.Ilu(A, oracle.ILUT, tau=1e-3, lfil=10)
    assert f.L.nnz == 0
    f = oracle.Ilu(A, oracle.ILUT, tau=1e-7, lfil=10)
    assert f.L.nnz == 1 and f.L[1, 0] == pytest.approx(1e-6)


def _csr(rows, n):
    M = np.zeros((n, n))
    for i, r in enumerate(rows):
        for j, v in r.items():
            M[i, j] = v
    return sp.csr_matrix(M)


def test_ilut_keeps_the_lfil_largest_with_ties_to_smaller_column():
    """Saad's ILUT (reading Q9) keeps the lfil LARGEST |w_j| of the L part
    and of the U part, ties to the smaller column — hand-computed rows where the largest
    are not the first columns (identity rows elsewhere: no elimination, no fill)."""
    lo = _csr([{0: 1}, {1: 1}, {2: 1}, {3: 1}, {0: 0.1, 1: 0.5, 2: -0.3, 3: -0.5, 4: 1}], 5)
    for lfil, keep in ((1, [1]), (2, [1, 3]), (3, [1, 2, 3]), (4, [0, 1, 2, 3])):
        f = oracle.Ilu(lo, oracle.ILUT, tau=1e-3, lfil=lfil)
        L = f.L.toarray()
        assert sorted(np.nonzero(L[4])[0].tolist()) == keep, (lfil, L[4])
        assert np.array_equal(L[4, keep], lo.toarray()[4, keep])
        assert np.array_equal(f.U.toarray(), np.eye(5))
    up = _csr([{0: 1, 1: 0.2, 2: -0.7, 3: 0.7, 4: 0.4}, {1: 1}, {2: 1}, {3: 1}, {4: 1}], 5)
    for lfil, keep in ((1, [0, 2]), (2, [0, 2, 3]), (3, [0, 2, 3, 4])):
        f = oracle.Ilu(up, oracle.ILUT, tau=1e-3, lfil=lfil)
        U = f.U.toarray()
        assert sorted(np.nonzero(U[0])[0].tolist()) == keep, (lfil, U[0])
        assert np.array_equal(U[0, keep], up.toarray()[0, keep])
        assert f.L.nnz == 0


def test_ilut_selects_after_elimination():
    """The lfil selection acts on the eliminated row w (Saad's order, reading Q9): a dropped
    L multiplier still updated the row before it was dropped.  Hand-computed:
    row 2 = [1, 0.6, 4]: w_0 = 1/2 = 0.5 (then w_2 = 4 - 0.5*3 = 2.5), w_1 = 0.6;
    lfil = 1 keeps l_21 = 0.6 (the larger, not the first), u_22 = 2.5."""
    A = _csr([{0: 2, 2: 3}, {1: 1}, {0: 1, 1: 0.6, 2: 4}], 3)
    f = oracle.Ilu(A, oracle.ILUT, tau=1e-3, lfil=1)
    assert np.array_equal(f.L.toarray(), np.array([[0, 0, 0], [0, 0, 0], [0, 0.6, 0]]))
    assert np.array_equal(f.U.toarray(), np.array([[2, 0, 3], [0, 1, 0], [0, 0, 2.5]]))
    f = oracle.Ilu(A, oracle.ILUT, tau=1e-3, lfil=2)             # both kept: exact LU
    assert np.abs(((f.L + sp.identity(3)) @ f.U - A).toarray()).max() < 1e-15


# ---------------------------------------------------------------- apply (c4)
def _exact_precond(prob, levels, p):
    A = prob.scipy()
    st = D.tiny_structure(A, prob.coords, levels, p, nlast=1)
    Pc = oracle.Precond(A, st, ilu=(oracle.ILUT, 0.0, 10**6))
    L = len(st["level_off"]) - 1
    for l in range(L - 1, -1, -1):       # bottom-up
        W, R, G = D.lowrank_from_dense(D.dense_ghat(Pc, l), k=None)
        Pc.set_lowrank(l, W, G)
    return A, st, Pc


@pytest.mark.parametrize("kind,dims,levels,p", [("lap", (8, 8), 1, 4), ("lap", (12, 12), 2, 4),
                                                ("cd", (6, 6, 4), 2, 4), ("hz", (5, 5, 4), 2, 2)])
def test_exact_mode_apply_is_inverse_D2(kind, dims, levels, p):
    prob = {"lap": P.laplacian, "cd": P.convdiff_upwind, "hz": P.helmholtz_shifted}[kind](dims)
    A, st, Pc = _exact_precond(prob, levels, p)
    Ah = D.permute_matrix(A, st["perm"]).toarray()
    b = P.rhs_vector(prob.n, prob.is_complex, 7)
    y = Pc.apply(b)
    ref = np.linalg.solve(Ah, b)
    assert np.linalg.norm(y - ref) <= 1e-10 * np.linalg.norm(ref)
    # natural-order form P M^{-1} Pᵀ = A^{-1}
    yn = Pc.apply_natural(b)
    refn = np.linalg.solve(A.toarray(), b)
    assert np.linalg.norm(yn - refn) <= 1e-10 * np.linalg.norm(refn)


def _rand_unitary(s, cplx, seed):
    r = rng(seed)
    M = r.standard_normal((s, s)) + (1j * r.standard_normal((s, s)) if cplx else 0)
    Q, _ = np.linalg.qr(M)
    return Q


@pytest.mark.parametrize("kind,dims,levels,p", [("hz", (5, 5, 4), 2, 2), ("hz", (8, 7), 1, 4),
                                                ("cd", (6, 6, 4), 2, 4)])
def test_exact_mode_rotated_basis_D2(kind, dims, levels, p):
    """Exact mode with W = Q, a random unitary (orthogonal for real A), and R = Q^H Ĝ Q:
    the correction W[(I-R)^{-1} - I]W^H = (I - Ĝ)^{-1} - I is basis-invariant
    (P:L401-404), so the apply is still Â^{-1}.  With a non-identity complex W a missing
    conjugate in s = W^H z2, or a transposed W or G, breaks the identity (W = I hides it).
    The same for the root preconditioner P = C_0^{-1}(I + W_0 G_0 W_0^H) = Ŝ_0^{-1} of
    NEXT-1 (lowrank_add): one root GMRES step is then exact."""
    prob = {"cd": P.convdiff_upwind, "hz": P.helmholtz_shifted}[kind](dims)
    A = prob.scipy()
    st = D.tiny_structure(A, prob.coords, levels, p, nlast=1)
    Pc = oracle.Precond(A, st, ilu=(oracle.ILUT, 0.0, 10**6))
    L = len(st["level_off"]) - 1
    for l in range(L - 1, -1, -1):
        Gm = D.dense_ghat(Pc, l)
        Q = _rand_unitary(Gm.shape[0], prob.is_complex, 40 + l)
        assert np.abs(Q - np.eye(Gm.shape[0])).max() > 0.1
        I = np.eye(Gm.shape[0])
        R = Q.conj().T @ Gm @ Q
        Pc.set_lowrank(l, Q, np.linalg.inv(I - R) - I)
    Ah = D.permute_matrix(A, st["perm"]).toarray()
    b = P.rhs_vector(prob.n, prob.is_complex, 7)
    ref = np.linalg.solve(Ah, b)
    assert np.linalg.norm(Pc.apply(b) - ref) <= 1e-10 * np.linalg.norm(ref)
    Pc.set_root_its(1)
    assert np.linalg.norm(Pc.apply(b) - ref) <= 1e-10 * np.linalg.norm(ref)


def test_ilu0_fullrank_is_exact_on_interface_D2():
    # 1 level, p = 2 on a 2D grid: the separator is one grid line, so C is
    # tridiagonal in index order and its ILU(0) is its exact LU (D8).  With a
    # full-rank correction the interface part of the apply is then Ŝ^{-1} z2,
    # Ŝ = C - E (LU)^{-1} F ("exact inverse on the interface").
    prob = P.convdiff_upwind((10, 10))
    A = prob.scipy()
    st = D.tiny_structure(A, prob.coords, 1, 2, nlast=1)
    Pc = oracle.Precond(A, st, ilu=(oracle.ILU0, 0.0, 0))
    W, R, G = D.lowrank_from_dense(D.dense_ghat(Pc, 0), k=None)
    Pc.set_lowrank(0, W, G)
    Ah = D.permute_matrix(A, st["perm"]).toarray()
    o1 = st["level_off"][1]
    Fm, Em, Cm = Ah[:o1, o1:], Ah[o1:, :o1], Ah[o1:, o1:]
    assert np.count_nonzero(np.triu(Cm, 2)) == 0          # tridiagonal C
    LUinv = np.zeros((o1, o1))
    bl = st["blocks"][0]
    for q in range(len(bl) - 1):
        a, c = bl[q], bl[q + 1]
        LUinv[a:c, a:c] = np.linalg.inv((Pc.factor(0, q, 0).toarray() + np.eye(c - a)) @ Pc.factor(0, q, 1).toarray())
    Shat = Cm - Em @ LUinv @ Fm
    b = P.rhs_vector(prob.n, False, 3)
    z1 = LUinv @ b[:o1]
    z2 = b[o1:] - Em @ z1
    y2 = np.linalg.solve(Shat, z2)
    y1 = z1 - LUinv @ Fm @ y2
    ref = np.concatenate([y1, y2])
    y = Pc.apply(b)
    assert np.linalg.norm(y - ref) <= 1e-10 * np.linalg.norm(ref)


def test_k0_apply_is_block_ldu_D5():
    prob = P.convdiff_upwind((9, 9))
    A = prob.scipy()
    st = D.tiny_structure(A, prob.coords, 1, 4, nlast=3)
    Pc = oracle.Precond(A, st, ilu=(oracle.ILU0, 0.0, 0))
    Ah = D.permute_matrix(A, st["perm"]).toarray()
    o1 = st["level_off"][1]
    n = prob.n
    LUinv = np.zeros((o1, o1))
    bl = st["blocks"][0]
    for q in range(len(bl) - 1):
        a, c = bl[q], bl[q + 1]
        LUinv[a:c, a:c] = np.linalg.inv((Pc.factor(0, q, 0).toarray() + np.eye(c - a)) @ Pc.factor(0, q, 1).toarray())
    Cinv = np.zeros((n - o1, n - o1))
    lo = st["last_off"] - o1
    for q in range(len(lo) - 1):
        a, c = lo[q], lo[q + 1]
        Cinv[a:c, a:c] = np.linalg.inv((Pc.factor(1, q, 0).toarray() + np.eye(c - a)) @ Pc.factor(1, q, 1).toarray())
    Fm, Em = Ah[:o1, o1:], Ah[o1:, :o1]
    I1, I2 = np.eye(o1), np.eye(n - o1)
    Minv = (np.block([[I1, -LUinv @ Fm], [np.zeros((n - o1, o1)), I2]])
            @ sla.block_diag(LUinv, Cinv)
            @ np.block([[I1, np.zeros((o1, n - o1))], [-Em @ LUinv, I2]]))
    b = P.rhs_vector(n, False, 11)
    assert np.linalg.norm(Pc.apply(b) - Minv @ b) <= 1e-12 * np.linalg.norm(Minv @ b)


@pytest.mark.parametrize("shift", [0.05, 0.5])
def test_complex_shifted_ilu_NEXT3(shift):
    """Complex shift of the block ILUs: with exact factors (ILUT tau = 0,
    lfil = inf) every block's L U equals B + sigma I, sigma = i*shift*sum|a_ii|/n_A — the
    textbook LU of the shifted block — and shift 0 gives the unshifted factors."""
    prob = P.helmholtz_shifted((7, 6, 5))
    A = prob.scipy()
    st = D.tiny_structure(A, prob.coords, 1, 4, nlast=2)
    Ah = D.permute_matrix(A, st["perm"]).toarray()
    sigma = 1j * shift * np.abs(A.diagonal()).sum() / A.shape[0]
    Pc = oracle.Precond(A, st, ilu=(oracle.ILUT, 0.0, 1 << 30), shift=shift)
    blocks = [(0, q, st["blocks"][0]) for q in range(len(st["blocks"][0]) - 1)]
    blocks += [(1, q, st["last_off"]) for q in range(len(st["last_off"]) - 1)]
    for l, q, bl in blocks:
        a, c = bl[q], bl[q + 1]
        Lq = Pc.factor(l, q, 0).toarray() + np.eye(c - a)
        Uq = Pc.factor(l, q, 1).toarray()
        B = Ah[a:c, a:c] + sigma * np.eye(c - a)
        assert np.abs(Lq @ Uq - B).max() <= 1e-12 * np.abs(B).max()
    P0 = oracle.Precond(A, st, ilu=(oracle.ILU0, 0.0, 0), shift=0.0)
    P1 = oracle.Precond(A, st, ilu=(oracle.ILU0, 0.0, 0))
    r = P.rhs_vector(prob.n, True, 4)
    assert np.array_equal(P0.apply(r), P1.apply(r))


@pytest.mark.parametrize("cplx", [False, True])
def test_root_gmres_NEXT1(cplx):
    """Root-level inner GMRES on Ŝ_0 (Alg. 2 line 6): run to s_0 steps it solves
    Ŝ_0 y2 = z2 exactly, so the apply equals the exact inverse of the block matrix
    [[L U, F_0], [E_0, C_0]] built densely from the oracle's own block ILU(0) factors; the
    map is homogeneous (apply(2b) = 2 apply(b)) but, with few steps, not additive."""
    prob = P.helmholtz_shifted((8, 7)) if cplx else P.convdiff_upwind((9, 8))
    A = prob.scipy()
    st = D.tiny_structure(A, prob.coords, 2, 4, nlast=2)
    Pc = oracle.Precond(A, st, ilu=(oracle.ILU0, 0.0, 0))
    n, o1 = prob.n, st["level_off"][1]
    s0 = n - o1
    Pc.set_root_its(s0)
    Ah = D.permute_matrix(A, st["perm"]).toarray()
    LU = np.zeros((o1, o1), dtype=Ah.dtype)
    bl = st["blocks"][0]
    for q in range(len(bl) - 1):
        a, c = bl[q], bl[q + 1]
        LU[a:c, a:c] = (Pc.factor(0, q, 0).toarray() + np.eye(c - a)) @ Pc.factor(0, q, 1).toarray()
    M = Ah.copy()
    M[:o1, :o1] = LU
    b = P.rhs_vector(n, cplx, 7)
    y = Pc.apply(b)
    ye = np.linalg.solve(M, b)
    assert np.linalg.norm(y - ye) <= 1e-9 * np.linalg.norm(ye)
    Pc.set_root_its(3)
    y1 = Pc.apply(b)
    assert np.linalg.norm(Pc.apply(2.0 * b) - 2.0 * y1) <= 1e-12 * np.linalg.norm(y1)
    b2 = P.rhs_vector(n, cplx, 8)
    assert np.linalg.norm(Pc.apply(b + b2) - y1 - Pc.apply(b2)) > 1e-8 * np.linalg.norm(y1)
    Pc.set_root_its(0)
    assert np.linalg.norm(Pc.apply(b + b2) - Pc.apply(b) - Pc.apply(b2)) <= 1e-12 * np.linalg.norm(y1)


def test_apply_linearity_D6_and_ghat_definition():
    prob = P.helmholtz_shifted((6, 6, 3))
    A = prob.scipy()
    st = D.tiny_structure(A, prob.coords, 2, 2, nlast=2)
    Pc = oracle.Precond(A, st, ilu=(oracle.ILUT, 1e-2, 3))
    r = rng(8)
    for l in range(len(st["level_off"]) - 2, -1, -1):
        Gm = D.dense_ghat(Pc, l)
        W, R, G = D.lowrank_from_dense(Gm, k=3)
        Pc.set_lowrank(l, W, G)
    a = P.rhs_vector(prob.n, True, 1)
    b = P.rhs_vector(prob.n, True, 2)
    al = 0.3 - 0.7j
    lhs = Pc.apply(al * a + b)
    rhs = al * Pc.apply(a) + Pc.apply(b)
    assert np.linalg.norm(lhs - rhs) <= 1e-12 * np.linalg.norm(rhs)
    assert np.all(Pc.apply(np.zeros(prob.n, complex)) == 0)
    # Ĝ_0 against its definition E (LU)^{-1} F C_0^{-1}, C_0^{-1} = apply from level 1
    o = st["level_off"]
    Ah = D.permute_matrix(A, st["perm"]).toarray()
    v = r.uniform(-1, 1, Pc.s(0)) + 1j * r.uniform(-1, 1, Pc.s(0))
    # C_0^{-1} v via apply_from(1) on the suffix
    cinv = Pc.apply(v, l0=1)
    bl = st["blocks"][0]
    LUinv = np.zeros((o[1], o[1]), complex)
    for q in range(len(bl) - 1):
        s0, s1 = bl[q], bl[q + 1]
        LUinv[s0:s1, s0:s1] = np.linalg.inv((Pc.factor(0, q, 0).toarray() + np.eye(s1 - s0)) @ Pc.factor(0, q, 1).toarray())
    ref = Ah[o[1]:, :o[1]] @ (LUinv @ (Ah[:o[1], o[1]:] @ cinv))
    assert np.linalg.norm(Pc.ghat(0, v) - ref) <= 1e-12 * np.linalg.norm(ref)


# ---------------------------------------------------------------- low rank closed forms
@pytest.mark.parametrize("seed", range(20))
def test_smw_identity_D3(seed):
    r = rng(100 + seed)
    nb, s = r.integers(5, 20), r.integers(3, 20)
    n = nb + s
    M = r.standard_normal((n, n)) + 1j * r.standard_normal((n, n)) + 3 * n * np.eye(n)
    Bm, Fm, Em, Cm = M[:nb, :nb], M[:nb, nb:], M[nb:, :nb], M[nb:, nb:]
    Gm = Em @ np.linalg.solve(Bm, Fm) @ np.linalg.inv(Cm)       # G = E B^-1 F C^-1
    T, Z = sla.schur(Gm, output="complex")                        # G = W R W^H
    S = Cm - Em @ np.linalg.solve(Bm, Fm)
    Sinv = np.linalg.inv(S)
    assert np.linalg.norm(Sinv - D.smw_inverse(Cm, Z, T)) <= 1e-10 * np.linalg.norm(Sinv)


def test_eigen_map_D4():
    r = rng(9)
    s = 12
    Gm = 0.5 * (r.standard_normal((s, s)) + 1j * r.standard_normal((s, s))) / np.sqrt(s)
    W, R, G = D.lowrank_from_dense(Gm, k=None)
    T, Z = sla.schur(Gm, output="complex")
    I = np.eye(s)
    corr = Z @ (np.linalg.inv(I - T) - I) @ Z.conj().T
    gam = np.linalg.eigvals(Gm)
    ev = np.linalg.eigvals(corr)
    exp = gam / (1 - gam)
    for e in exp:
        assert np.min(np.abs(ev - e)) <= 1e-8 * max(1, abs(e))


def test_partial_rank_real_schur_keeps_pairs():
    r = rng(10)
    Gm = r.standard_normal((15, 15)) / 5
    W, R, G = D.lowrank_from_dense(Gm, k=4)
    assert W.dtype == np.float64 and W.shape[1] in (4, 5)
    assert np.abs(W.T @ W - np.eye(W.shape[1])).max() < 1e-12
    assert np.abs(W.T @ Gm @ W - R).max() < 1e-12


# ---------------------------------------------------------------- FGMRES (c5)
def test_fgmres_identity_one_iteration_D7():
    A = sp.identity(30, format="csr")
    b = rng(11).uniform(-1, 1, 30)
    out = oracle.fgmres(A, b, rtol=1e-10, restart=10)
    assert out["its"] == 1 and np.allclose(out["x"], b, atol=1e-14)


@pytest.mark.parametrize("cplx", [False, True])
def test_fgmres_exact_preconditioner_one_iteration_D7(cplx):
    prob = P.helmholtz_shifted((5, 4, 3)) if cplx else P.convdiff_upwind((6, 5))
    A = prob.scipy()
    Ad = A.toarray()
    b = P.rhs_vector(prob.n, cplx, 4)
    out = oracle.fgmres(A, b, M=lambda v: np.linalg.solve(Ad, v), rtol=1e-10, restart=10)
    assert out["its"] == 1
    assert np.linalg.norm(Ad @ out["x"] - b) <= 1e-10 * np.linalg.norm(b)


@pytest.mark.parametrize("cplx", [False, True])
def test_fgmres_dense_direct_solve_D1(cplx):
    prob = P.helmholtz_shifted((6, 6, 4)) if cplx else P.laplacian((32, 32))
    A = prob.scipy()
    b = P.rhs_vector(prob.n, cplx, 0)
    rtol = 1e-8
    out = oracle.fgmres(A, b, rtol=rtol, restart=30, maxit=3000, diag=True)
    assert out["status"] == 0
    Ad = A.toarray()
    xs = np.linalg.solve(Ad, b)
    assert np.linalg.norm(Ad @ out["x"] - b) <= rtol * np.linalg.norm(b)
    assert out["final_relres"] <= rtol
    kappa = np.linalg.cond(Ad)
    assert np.linalg.norm(out["x"] - xs) <= kappa * rtol * np.linalg.norm(xs)
    assert out["orth"] <= 1e-12           # ||V^H V - I||_max, CGS2 (Q14)
    assert out["arnoldi"] <= 1e-12        # ||A Z - V Hbar||_F / (||A||_F ||Z||_F)
    assert out["est_gap"] <= 1e-8         # Givens estimate vs explicit residual
    assert out["hist"][0] == pytest.approx(1.0)
    assert np.all(np.diff(out["hist"][:31]) <= 1e-15)   # monotone within the first cycle


# ---------------------------------------------------------------- FGMRES with DCGS2 (c5', Q38)
def test_fgmres_dcgs2_identity_and_exact_preconditioner_one_iteration_D7():
    A = sp.identity(30, format="csr")
    b = rng(11).uniform(-1, 1, 30)
    out = oracle.fgmres(A, b, rtol=1e-10, restart=10, orth="dcgs2")
    assert out["its"] == 1 and np.allclose(out["x"], b, atol=1e-14)
    for cplx in (False, True):
        prob = P.helmholtz_shifted((5, 4, 3)) if cplx else P.convdiff_upwind((6, 5))
        Ad = prob.scipy().toarray()
        b = P.rhs_vector(prob.n, cplx, 4)
        out = oracle.fgmres(prob.scipy(), b, M=lambda v: np.linalg.solve(Ad, v), rtol=1e-10, restart=10,
                            orth="dcgs2")
        assert out["its"] == 1
        assert np.linalg.norm(Ad @ out["x"] - b) <= 1e-10 * np.linalg.norm(b)


@pytest.mark.parametrize("cplx", [False, True])
def test_fgmres_dcgs2_dense_direct_solve_D1(cplx):
    """The same closed-form checks as CGS2 (D1): solution against a dense solve, VᴴV = I and
    the Arnoldi relation A Z = V H̄ to 1e-12 (north_star), estimate = explicit residual."""
    prob = P.helmholtz_shifted((6, 6, 4)) if cplx else P.laplacian((32, 32))
    A = prob.scipy()
    b = P.rhs_vector(prob.n, cplx, 0)
    rtol = 1e-8
    out = oracle.fgmres(A, b, rtol=rtol, restart=30, maxit=3000, diag=True, orth="dcgs2")
    assert out["status"] == 0
    Ad = A.toarray()
    xs = np.linalg.solve(Ad, b)
    assert np.linalg.norm(Ad @ out["x"] - b) <= rtol * np.linalg.norm(b)
    kappa = np.linalg.cond(Ad)
    assert np.linalg.norm(out["x"] - xs) <= kappa * rtol * np.linalg.norm(xs)
    assert out["orth"] <= 1e-12
    assert out["arnoldi"] <= 1e-12
    assert out["est_gap"] <= 1e-8
    assert out["hist"][0] == pytest.approx(1.0)
    assert np.all(np.diff(out["hist"][:31]) <= 1e-15)


@pytest.mark.parametrize("cplx", [False, True])
@pytest.mark.parametrize("orth", ["cgs2", "dcgs2"])
def test_fgmres_history_is_the_least_squares_minimum_over_span_Z(cplx, orth):
    """FGMRES: after k columns the residual estimate is
    min_y ||b - A Z_k y|| / ||b||, Z_k the preconditioned vectors (any scaling: the span
    counts).  A preconditioner that changes at every call (flexible) is recorded and the
    minimum is recomputed by a dense least-squares solve — a dropped term, a sign or a
    missing conjugate in the Hessenberg columns breaks the equality."""
    prob = P.helmholtz_shifted((5, 4, 4)) if cplx else P.convdiff_upwind((9, 8))
    A = prob.scipy()
    Ad = A.toarray()
    n = prob.n
    b = P.rhs_vector(n, cplx, 6)
    r = rng(21)
    Zs = []

    def M(v):                     # a different diagonal scaling at every call: flexible
        d = 1.0 / (np.diag(Ad) * (1.0 + 0.5 * r.uniform(-1, 1, n)))
        z = d * v
        Zs.append(z.copy())
        return z

    m = 12
    out = oracle.fgmres(A, b, M=M, rtol=1e-300, restart=m, maxit=m, orth=orth)
    assert out["its"] == m
    Z = np.array(Zs[:m]).T
    bn = np.linalg.norm(b)
    for k in range(1, m + 1):
        AZ = Ad @ Z[:, :k]
        y, *_ = np.linalg.lstsq(AZ, b, rcond=None)
        best = np.linalg.norm(b - AZ @ y) / bn
        assert out["hist"][k] == pytest.approx(best, rel=1e-7, abs=1e-14), (k, out["hist"][k], best)
    x_ref = Z @ np.linalg.lstsq(Ad @ Z, b, rcond=None)[0]
    assert np.linalg.norm(out["x"] - x_ref) <= 1e-8 * np.linalg.norm(x_ref)


@pytest.mark.parametrize("cplx", [False, True])
@pytest.mark.parametrize("orth", ["cgs2", "dcgs2"])
def test_fgmres_orthonormal_basis_on_an_ill_conditioned_krylov_sequence(cplx, orth):
    """north_star: ||VᴴV − I|| <= 1e-12.  Eigenvalues spread over 8 decades make the
    Krylov vectors nearly dependent; one Gram–Schmidt pass then leaves ~1e-12 and worse,
    the second (immediate in CGS2, delayed in DCGS2) brings it back to ~1e-15."""
    n = 400
    r = rng(3)
    ev = np.logspace(-8, 0, n)
    if cplx:
        ev = ev * np.exp(1j * r.uniform(0, 0.3, n))
    A = sp.diags([ev, 0.3 * ev[:-1]], [0, 1], format="csr")
    b = r.uniform(-1, 1, n) + (1j * r.uniform(-1, 1, n) if cplx else 0)
    out = oracle.fgmres(A, b, rtol=1e-300, restart=80, maxit=80, diag=True, orth=orth)
    assert out["its"] == 80
    assert out["orth"] <= 2e-14
    assert out["arnoldi"] <= 1e-14


def test_fgmres_dcgs2_matches_cgs2_iterations_with_gemslr():
    """Both orthogonalisations are CGS applied twice; with the GeMSLR oracle as the
    preconditioner they need the same number of iterations (±1) and reach rtol."""
    prob = P.laplacian((16, 16, 8))
    A = prob.scipy()
    b = P.rhs_vector(prob.n, False, 0)
    st = D.tiny_structure(A, prob.coords, 2, 4, nlast=4)
    Pc = oracle.Precond(A, st, ilu=(oracle.ILUT, 1e-3, 10))
    o1 = oracle.fgmres(A, b, M=Pc, rtol=1e-8, restart=20)
    o2 = oracle.fgmres(A, b, M=Pc, rtol=1e-8, restart=20, orth="dcgs2")
    assert o1["status"] == 0 and o2["status"] == 0
    assert abs(o1["its"] - o2["its"]) <= 1
    assert np.linalg.norm(A @ o2["x"] - b) <= 1e-8 * np.linalg.norm(b)
    k = min(len(o1["hist"]), len(o2["hist"]))
    assert np.allclose(o1["hist"][:k], o2["hist"][:k], rtol=1e-6, atol=1e-13)


def test_fgmres_with_gemslr_oracle_converges_and_rank_helps():
    prob = P.laplacian((16, 16, 8))
    A = prob.scipy()
    b = P.rhs_vector(prob.n, False, 0)
    st = D.tiny_structure(A, prob.coords, 2, 4, nlast=4)
    its = []
    for k in (0, 6):
        Pc = oracle.Precond(A, st, ilu=(oracle.ILUT, 1e-3, 10))
        if k:
            for l in range(len(st["level_off"]) - 2, -1, -1):
                W, R, G = D.lowrank_from_dense(D.dense_ghat(Pc, l), k=k)
                Pc.set_lowrank(l, W, G)
        out = oracle.fgmres(A, b, M=Pc, rtol=1e-8, restart=50)
        assert out["status"] == 0
        assert np.linalg.norm(A @ out["x"] - b) <= 1e-8 * np.linalg.norm(b)
        its.append(out["its"])
    assert its[1] <= its[0]                # S:L490 soft check


def test_oracle_results_do_not_depend_on_thread_count():
    """the OpenMP oracle sums in fixed chunks, so 1 and 4 threads give
    bit-identical applies and FGMRES histories (vectors longer than one chunk)."""
    prob = P.laplacian((24, 24, 24))
    A = prob.scipy()
    st = D.tiny_structure(A, prob.coords, 2, 8, nlast=4)
    b = P.rhs_vector(prob.n, False, 3)
    res = []
    nt0 = oracle.get_threads()
    try:
        for nt in (1, 4):
            oracle.set_threads(nt)
            Pc = oracle.Precond(A, st, ilu=(oracle.ILUT, 1e-3, 10))
            out = oracle.fgmres(prob, b, M=Pc, rtol=1e-10, restart=20)
            res.append((Pc.apply(b), out["x"], out["hist"]))
    finally:
        oracle.set_threads(nt0)
    for a, c in zip(res[0], res[1]):
        assert np.array_equal(a, c)
