"""GPU parity: the CUDA path (through the C-ABI) against the independent oracle.

Bar (BASELINE.json north_star): ||y_gpu - y_or||_2 <= 1e-10 ||y_or||_2
on every SpMV and preconditioner application (fp64 and complex128); FGMRES
iteration count within ±1 of the oracle's; final true residual <= rtol.

The setup is non-unique (partition ties, Arnoldi subspaces), so both sides
consume ONE exported bundle: the oracle verifies it independently (c3) — its
own Â from its own A, its own ILU factors recomputed and compared, W
orthonormal, the Rayleigh quotient W^H Ĝ W ≈ R with its own Ĝ, the identity
(I - R)(G + I) = I — and then runs its own apply with its own factors and the
bundle's W, G.
"""
import numpy as np
import pytest

import oracle
from oracle import dense as D
from synth import problems as P
from tests.bundle_io import Bundle

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
gm = pytest.importorskip("paper_2205_03224_b200")

TOL = 1e-10


def rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def make_pair(prob, prm, tmp_path, coords=True, **kw):
    """GPU solver + oracle preconditioner on the same verified bundle."""
    s = gm.Solver(prob.rowptr, prob.colidx, prob.values, prm["levels"], prm["subdomains"], prm["rank"],
                  ilu=prm["ilu"], ilut_drop=prm.get("ilut_drop", 1e-3), ilut_fill=prm.get("ilut_fill", 10),
                  coords=prob.coords if coords else None, device=0, **kw)
    d = s.export(str(tmp_path / "bundle"))
    B = Bundle(d)
    st = B.structure()
    A = prob.scipy()
    kind = oracle.ILU0 if prm["ilu"] == "ilu0" else oracle.ILUT
    Pc = oracle.Precond(A, st, ilu=(kind, prm.get("ilut_drop", 1e-3), prm.get("ilut_fill", 10)))
    for l in range(B.L):
        lr = B.lowrank(l)
        if lr is not None:
            W, R, G = lr
            Pc.set_lowrank(l, W, G)
    return s, B, st, Pc


def to_dev(s, v):
    return torch.from_numpy(np.ascontiguousarray(v)).to(device="cuda:0", dtype=s.torch_dtype)


def verify_lowrank(B, Pc, rank):
    for l in range(B.L):
        lr = B.lowrank(l)
        if lr is None:
            assert rank == 0 or Pc.s(l) == 0
            continue
        W, R, G = lr
        k = W.shape[1]
        assert rank <= k <= rank + 1 or k == Pc.s(l)
        assert np.abs(W.conj().T @ W - np.eye(k)).max() <= 1e-12            # c3.5
        GW = np.stack([Pc.ghat(l, W[:, c]) for c in range(k)], axis=1)
        WGW = W.conj().T @ GW
        assert np.linalg.norm(WGW - R) <= 1e-2 * np.linalg.norm(R)          # c3.6 Rayleigh
        I = np.eye(k)
        assert np.abs((I - R) @ (G + I) - I).max() <= 1e-12                 # c3.8


CASES = [
    ("C1", None, {}),
    ("C2", (20, 20, 20), dict(subdomains=8, rank=6)),
    ("C3", (20, 18, 16), dict(subdomains=8, rank=8)),
    ("C4", (16, 16, 14), dict(subdomains=8, rank=8)),
    ("C5", (24, 24, 24), dict(subdomains=8, rank=6)),
]


@pytest.mark.parametrize("name,dims,over", CASES)
def test_spmv_and_apply_parity(tmp_path, name, dims, over):
    prob, b, xt, prm = P.make_config(name, dims=dims, **over)
    s, B, st, Pc = make_pair(prob, prm, tmp_path)
    verify_lowrank(B, Pc, prm["rank"])
    perm = st["perm"]
    n = prob.n
    # SpMV: local permuted layout in, gathered back to natural order
    x = P.rhs_vector(n, prob.is_complex, 3)
    y = s.spmv(to_dev(s, x[perm])).cpu().numpy()
    ynat = np.empty_like(y)
    ynat[perm] = y
    assert rel(ynat, oracle.spmv(prob, x)) <= TOL
    # apply: several vectors, incl. structured ones
    for seed, scale in ((5, 1.0), (6, 1e-3), (7, 1e5)):
        r = P.rhs_vector(n, prob.is_complex, seed) * scale
        yg = s.apply_precond(to_dev(s, r)).cpu().numpy()
        yo = Pc.apply(r)
        assert rel(yg, yo) <= TOL, (seed, rel(yg, yo))
    e = np.zeros(n, dtype=prob.values.dtype)
    e[n // 2] = 1
    assert rel(s.apply_precond(to_dev(s, e)).cpu().numpy(), Pc.apply(e)) <= TOL
    z = s.apply_precond(to_dev(s, np.zeros(n, dtype=prob.values.dtype))).cpu().numpy()
    assert np.all(z == 0)


@pytest.mark.parametrize("name,dims,over", CASES)
def test_solve_parity(tmp_path, name, dims, over):
    prob, b, xt, prm = P.make_config(name, dims=dims, **over)
    s, B, st, Pc = make_pair(prob, prm, tmp_path)
    perm = st["perm"]
    out = s.solve(to_dev(s, b[perm]), rtol=prm["rtol"], restart=prm["restart"], maxit=1000)
    xg = np.empty(prob.n, dtype=prob.values.dtype)
    xg[perm] = out["x"].cpu().numpy()
    ref = oracle.fgmres(prob, b, M=Pc, rtol=prm["rtol"], restart=prm["restart"], maxit=1000)
    assert out["status"] == 0 and ref["status"] == 0
    assert abs(out["its"] - ref["its"]) <= 1, (out["its"], ref["its"])
    true_rel = np.linalg.norm(b - oracle.spmv(prob, xg)) / np.linalg.norm(b)
    assert true_rel <= prm["rtol"]
    assert out["final_relres"] == pytest.approx(true_rel, rel=1e-6, abs=1e-14)
    # residual histories agree while above the rounding floor
    h = min(len(out["hist"]), len(ref["hist"]))
    assert np.allclose(out["hist"][:h], ref["hist"][:h], rtol=1e-6, atol=1e2 * prm["rtol"])
    if xt is not None:
        assert np.linalg.norm(xg - xt) <= 1e3 * prm["rtol"] * np.linalg.norm(xt)


def test_solve_host_path_matches_device_path(tmp_path):
    prob, b, xt, prm = P.make_config("C2", dims=(16, 16, 16), subdomains=8, rank=6)
    s, B, st, Pc = make_pair(prob, prm, tmp_path)
    perm = st["perm"]
    dev = s.solve(to_dev(s, b[perm]), rtol=prm["rtol"], restart=prm["restart"])
    host = s.solve_host(b, rtol=prm["rtol"], restart=prm["restart"])
    xd = np.empty(prob.n)
    xd[perm] = dev["x"].cpu().numpy()
    assert host["its"] == dev["its"]
    assert rel(host["x"], xd) <= 1e-13
    # to_local / to_natural round trip
    v = to_dev(s, P.rhs_vector(prob.n, False, 1))
    assert torch.equal(s.to_natural(s.to_local(v)), v)


def test_dense_spectrum_C1(tmp_path):
    """c3.7: on C1 the selected Ritz values match, to two digits, the k eigenvalues of
    the dense Ĝ_0 with the largest |γ/(1-γ)|."""
    prob, b, xt, prm = P.make_config("C1")
    s, B, st, Pc = make_pair(prob, prm, tmp_path)
    W, R, G = B.lowrank(0)
    Gm = D.dense_ghat(Pc, 0)
    ev = np.linalg.eigvals(Gm)
    key = np.abs(ev / (1 - ev))
    top = ev[np.argsort(-key)][:W.shape[1]]
    ritz = np.linalg.eigvals(R)
    for t in top[:prm["rank"] - 1]:
        assert np.min(np.abs(ritz - t)) <= 1e-2 * max(abs(t), 1e-3)


def test_rank_zero_and_ilu0_variants(tmp_path):
    prob, b, xt, prm = P.make_config("C3", dims=(14, 14, 14), subdomains=8, rank=0, ilu="ilu0")
    s, B, st, Pc = make_pair(prob, prm, tmp_path)
    r = P.rhs_vector(prob.n, False, 9)
    assert rel(s.apply_precond(to_dev(s, r)).cpu().numpy(), Pc.apply(r)) <= TOL


@pytest.mark.parametrize("cps", [1, 2, 4])
def test_cluster_sizes_agree(tmp_path, cps):
    prob, b, xt, prm = P.make_config("C5", dims=(32, 32, 32), subdomains=4, rank=4)
    s, B, st, Pc = make_pair(prob, prm, tmp_path, cluster_ctas=cps)
    r = P.rhs_vector(prob.n, False, 2)
    assert rel(s.apply_precond(to_dev(s, r)).cpu().numpy(), Pc.apply(r)) <= TOL


@pytest.mark.parametrize("name,dims,over", [("C5", (32, 32, 24), dict(subdomains=4, rank=4)),
                                             ("C4", (16, 16, 14), dict(subdomains=8, rank=6)),
                                             ("C3", (20, 18, 16), dict(subdomains=8, rank=0, ilu="ilu0"))])
@pytest.mark.parametrize("tri_kernel,expect", [(0, "reg"), (1, "pipe"), (2, "level")])
def test_trisolve_kernels(tmp_path, name, dims, over, tri_kernel, expect):
    """Each triangular-solve kernel (register-prefetched k_tri_reg, TMA-staged
    k_tri_pipe, level kernel) against the oracle, fp64 and complex128."""
    prob, b, xt, prm = P.make_config(name, dims=dims, **over)
    s, B, st, Pc = make_pair(prob, prm, tmp_path, tri_kernel=tri_kernel)
    assert all(L["stage"]["kernel"] == expect for L in s.stats()["stages"])
    for seed in (2, 3):
        r = P.rhs_vector(prob.n, prob.is_complex, seed)
        assert rel(s.apply_precond(to_dev(s, r)).cpu().numpy(), Pc.apply(r)) <= TOL


@pytest.mark.parametrize("name,dims,over", [("C5", (24, 24, 20), dict(subdomains=8, rank=4)),
                                             ("C4", (16, 16, 14), dict(subdomains=8, rank=6))])
def test_multiple_rhs_NEXT4(tmp_path, name, dims, over):
    """Several right-hand sides: SpMV and apply on (nrhs, n) blocks, with a
    leading dimension larger than n and more columns than one launch takes, equal the
    oracle column by column."""
    prob, b, xt, prm = P.make_config(name, dims=dims, **over)
    s, B, st, Pc = make_pair(prob, prm, tmp_path)
    n = prob.n
    perm = st["perm"]
    for nr in (1, 3, 11):
        big = torch.zeros((nr, n + 37), dtype=s.torch_dtype, device="cuda:0")
        cols = [P.rhs_vector(n, prob.is_complex, 100 + c) for c in range(nr)]
        for c in range(nr):
            big[c, :n] = to_dev(s, cols[c])
        X = big[:, :n]
        Y = s.apply_precond_multi(X).cpu().numpy()
        for c in range(nr):
            assert rel(Y[c], Pc.apply(cols[c])) <= TOL, (nr, c)
        Ys = s.spmv_multi(X).cpu().numpy()
        for c in range(nr):
            ynat = np.empty(n, dtype=Ys.dtype)
            ynat[perm] = Ys[c]
            xnat = np.empty(n, dtype=Ys.dtype)
            xnat[perm] = cols[c]
            assert rel(ynat, oracle.spmv(prob, xnat)) <= TOL


@pytest.mark.parametrize("name,dims,over", [("C5", (24, 24, 20), dict(subdomains=8, rank=4)),
                                             ("C4", (16, 16, 14), dict(subdomains=8, rank=6)),
                                             ("C3", (20, 18, 16), dict(subdomains=8, rank=0))])
@pytest.mark.parametrize("split", [1, 2])
def test_root_gmres_NEXT1(tmp_path, name, dims, over, split):
    """Root-level inner GMRES on Ŝ_0 (Alg. 2 line 6, 3 steps as in P:L1073-1074): apply
    parity against the oracle's root GMRES, FGMRES iterations within ±1, true residual."""
    prob, b, xt, prm = P.make_config(name, dims=dims, **over)
    s, B, st, Pc = make_pair(prob, prm, tmp_path, root_inner_its=3, tri_split=split)
    Pc.set_root_its(3)
    for seed in (2, 3):
        r = P.rhs_vector(prob.n, prob.is_complex, seed)
        assert rel(s.apply_precond(to_dev(s, r)).cpu().numpy(), Pc.apply(r)) <= TOL
    for orth in ("cgs2", "dcgs2"):                  # (DCGS2: the outer level-0 pre-packing is off here)
        out = s.solve(to_dev(s, b[st["perm"]]), rtol=prm["rtol"], restart=prm["restart"], orth=orth)
        ref = oracle.fgmres(prob, b, M=Pc, rtol=prm["rtol"], restart=prm["restart"], orth=orth)
        assert out["status"] == 0 and abs(out["its"] - ref["its"]) <= 1, (orth, out["its"], ref["its"])
        xg = np.empty(prob.n, dtype=b.dtype)
        xg[st["perm"]] = out["x"].cpu().numpy()
        assert np.linalg.norm(b - oracle.spmv(prob, xg)) <= prm["rtol"] * np.linalg.norm(b)


def test_complex_shifted_ilu_NEXT3(tmp_path):
    """C4 recipe with the paper's complex ILU shift 0.05 i sum|a_ii|/n:
    apply parity against the oracle's own shifted factors, FGMRES iterations within ±1."""
    prob, b, xt, prm = P.make_config("C4", dims=(16, 16, 14), subdomains=8, rank=6)
    s = gm.Solver(prob.rowptr, prob.colidx, prob.values, prm["levels"], prm["subdomains"], prm["rank"],
                  ilu=prm["ilu"], coords=prob.coords, device=0, ilu_shift=0.05)
    d = s.export(str(tmp_path / "bundle"))
    B = Bundle(d)
    st = B.structure()
    Pc = oracle.Precond(prob.scipy(), st, ilu=(oracle.ILUT, 1e-3, 10), shift=0.05)
    for l in range(B.L):
        lr = B.lowrank(l)
        if lr is not None:
            Pc.set_lowrank(l, lr[0], lr[2])
    for seed in (2, 3):
        r = P.rhs_vector(prob.n, True, seed)
        assert rel(s.apply_precond(to_dev(s, r)).cpu().numpy(), Pc.apply(r)) <= TOL
    out = s.solve(to_dev(s, b[st["perm"]]), rtol=prm["rtol"], restart=prm["restart"])
    ref = oracle.fgmres(prob, b, M=Pc, rtol=prm["rtol"], restart=prm["restart"])
    assert out["status"] == 0 and abs(out["its"] - ref["its"]) <= 1, (out["its"], ref["its"])
    with pytest.raises(gm.GemslrError):                    # real problems have no complex shift
        p5, _, _, q5 = P.make_config("C5", dims=(8, 8, 8), subdomains=4, rank=2)
        gm.Solver(p5.rowptr, p5.colidx, p5.values, q5["levels"], q5["subdomains"], q5["rank"], ilu=q5["ilu"],
                  coords=p5.coords, device=0, ilu_shift=0.05)


# ---------------------------------------------------------------- edge cases
@pytest.mark.parametrize("kind", ["tiny1d", "p1", "fullrank", "early_stop", "random_bfs", "complex_bfs"])
def test_edge_cases(tmp_path, kind):
    import scipy.sparse as sp
    if kind == "tiny1d":               # 1D chain: ILU(0) is exact LU, separators are points
        n = 40
        A = sp.diags([-1.0 * np.ones(n - 1), 2.5 * np.ones(n), -1.2 * np.ones(n - 1)], [-1, 0, 1], format="csr")
        prob = P.Problem("1d", (n,), A.indptr.astype(np.int64), A.indices.astype(np.int32), A.data,
                         np.stack([np.arange(n), np.zeros(n), np.zeros(n)], 1).astype(float))
        prm = dict(levels=2, subdomains=2, rank=2, ilu="ilu0")
    elif kind == "p1":                 # one subdomain per level
        prob = P.laplacian((9, 8, 7))
        prm = dict(levels=2, subdomains=1, rank=3, ilu="ilut")
    elif kind == "fullrank":           # rank >= separator size
        prob = P.convdiff_upwind((10, 10))
        prm = dict(levels=1, subdomains=4, rank=40, ilu="ilu0")
    elif kind == "early_stop":         # more levels requested than the separators allow
        prob = P.laplacian((12, 12))
        prm = dict(levels=6, subdomains=4, rank=4, ilu="ilut")
    elif kind == "random_bfs":         # unstructured nonsymmetric pattern, BFS partitioner
        r = np.random.default_rng(3)
        n = 600
        M = sp.random(n, n, density=6.0 / n, random_state=4, format="csr")
        M = M + M.T.multiply(r.uniform(0.5, 1.5, (n, n)) > 1.2) + sp.identity(n) * 8.0
        M = sp.csr_matrix(M)
        M.sort_indices()
        prob = P.Problem("rnd", (n,), M.indptr.astype(np.int64), M.indices.astype(np.int32), M.data,
                         np.zeros((n, 3)))
        prm = dict(levels=2, subdomains=4, rank=4, ilu="ilut")
    else:                              # complex without coordinates
        prob = P.helmholtz_shifted((8, 7, 6))
        prm = dict(levels=2, subdomains=4, rank=5, ilu="ilut")
    prm.update(ilut_drop=1e-3, ilut_fill=10)
    coords = kind not in ("random_bfs", "complex_bfs")
    s, B, st, Pc = make_pair(prob, prm, tmp_path, coords=coords)
    n = prob.n
    x = P.rhs_vector(n, prob.is_complex, 2)
    assert rel(s.apply_precond(to_dev(s, x)).cpu().numpy(), Pc.apply(x)) <= TOL
    y = s.spmv(to_dev(s, x[st["perm"]])).cpu().numpy()
    yn = np.empty_like(y)
    yn[st["perm"]] = y
    assert rel(yn, oracle.spmv(prob, x)) <= TOL
    b = P.rhs_vector(n, prob.is_complex, 9)
    out = s.solve(to_dev(s, b[st["perm"]]), rtol=1e-8, restart=20, maxit=400)
    ref = oracle.fgmres(prob, b, M=Pc, rtol=1e-8, restart=20, maxit=400)
    assert abs(out["its"] - ref["its"]) <= 1 and out["status"] == ref["status"] == 0


def test_zero_rhs_and_maxit(tmp_path):
    prob, b, xt, prm = P.make_config("C2", dims=(10, 10, 10), subdomains=4, rank=3)
    s, B, st, Pc = make_pair(prob, prm, tmp_path)
    out = s.solve(to_dev(s, np.zeros(prob.n)), rtol=1e-8, restart=10)
    assert out["its"] == 0 and out["status"] == 0 and torch.count_nonzero(out["x"]) == 0
    out = s.solve(to_dev(s, b[st["perm"]]), rtol=1e-14, restart=5, maxit=7)
    assert out["its"] == 7 and out["status"] == 1            # NOT_CONVERGED
    assert len(out["hist"]) == 8


@pytest.mark.parametrize("restart,maxit", [(1, 6), (2, 7), (5, 1), (5, 3), (7, 21)])
def test_dcgs2_degenerate_cycles(tmp_path, restart, maxit):
    """DCGS2 (Q38) at the cycle edges: restart 1 (every step closes its cycle), a cycle cut
    by maxit before its end, maxit = 1, whole cycles; zero right-hand side — histories and
    iteration counts against the oracle's fgmres_dcgs2."""
    prob, b, xt, prm = P.make_config("C2", dims=(10, 10, 10), subdomains=4, rank=3)
    s, B, st, Pc = make_pair(prob, prm, tmp_path)
    out = s.solve(to_dev(s, np.zeros(prob.n)), rtol=1e-8, restart=restart, orth="dcgs2")
    assert out["its"] == 0 and out["status"] == 0 and torch.count_nonzero(out["x"]) == 0
    out = s.solve(to_dev(s, b[st["perm"]]), rtol=1e-300, restart=restart, maxit=maxit, orth="dcgs2")
    ref = oracle.fgmres(prob, b, M=Pc, rtol=1e-300, restart=restart, maxit=maxit, orth="dcgs2")
    assert out["its"] == ref["its"] == maxit and out["status"] == 1
    assert len(out["hist"]) == len(ref["hist"]) == maxit + 1
    h = np.asarray(ref["hist"])
    keep = h > 1e-10
    assert np.allclose(out["hist"][keep], h[keep], rtol=1e-7, atol=0)
    xg = np.empty(prob.n)
    xg[st["perm"]] = out["x"].cpu().numpy()
    assert rel(xg, ref["x"]) <= 1e-7


@pytest.mark.parametrize("orth", ["cgs2", "dcgs2"])
def test_solve_twice_with_growing_maxit(tmp_path, orth):
    """The FGMRES iteration graphs are captured once per (restart, basis, history buffer):
    a second solve with a larger maxit (a new history buffer) must re-capture them and
    report the full history (stale graphs wrote past the old buffer)."""
    prob, b, xt, prm = P.make_config("C5", dims=(24, 24, 20), subdomains=8, rank=4)
    s, B, st, Pc = make_pair(prob, prm, tmp_path)
    bd = to_dev(s, b[st["perm"]])
    first = s.solve(bd, rtol=1e-300, restart=10, maxit=5, orth=orth)
    assert first["its"] == 5 and len(first["hist"]) == 6
    for maxit in (37, 80):
        out = s.solve(bd, rtol=1e-300, restart=10, maxit=maxit, orth=orth)
        ref = oracle.fgmres(prob, b, M=Pc, rtol=1e-300, restart=10, maxit=maxit, orth=orth)
        assert out["its"] == maxit and len(out["hist"]) == maxit + 1
        h = np.asarray(ref["hist"])
        keep = h > 1e-10            # above the rounding floor (the tail form sums in another order, DESIGN 6b)
        assert np.allclose(out["hist"][keep], h[keep], rtol=1e-6, atol=0)
        assert np.allclose(first["hist"], out["hist"][:6], rtol=1e-12, atol=0)


@pytest.mark.parametrize("rank", [47, 51])
def test_rank_near_the_limit(tmp_path, rank):
    """k_ewx with 6 / 8 accumulators per warp (k up to 52 after the conjugate-pair rule):
    apply parity with the oracle; rank 52 is refused."""
    prob, b, xt, prm = P.make_config("C5", dims=(28, 28, 24), subdomains=4, rank=rank, levels=2)
    s, B, st, Pc = make_pair(prob, prm, tmp_path)
    ks = [x["k"] for x in s.stats()["stages"]]
    assert ks[0] >= rank
    for seed in (2, 3):
        r = P.rhs_vector(prob.n, False, seed)
        assert rel(s.apply_precond(to_dev(s, r)).cpu().numpy(), Pc.apply(r)) <= TOL
    with pytest.raises(gm.GemslrError):
        gm.Solver(prob.rowptr, prob.colidx, prob.values, 2, 4, 52, coords=prob.coords, device=0)


@pytest.mark.parametrize("cplx,restart", [(False, 50), (False, 100), (True, 64), (True, 100)])
def test_gram_schmidt_every_column_count(tmp_path, cplx, restart):
    """CGS2 (reading Q14) at 1..restart columns, i.e. every Gram-Schmidt kernel the solver
    dispatches by column count: fp64 k_gs2<8..32> (<= 32), k_gs<4,6> / k_gs<2,6> /
    k_gs2<48> (33-48), k_gs2h (49-64), k_gs<1,13> (65-100); complex k_gs2<8..32>,
    k_gs<2,6> (33-48), k_gs2g<2,32> (49-64), k_gs2g<4,26> (65-104).  The problem is
    indefinite (shifted Laplacian / weakly damped Helmholtz) so the residual stays well
    above the rounding floor through the whole cycle and every column's Hessenberg
    entries shape the history: histories equal the oracle's to 1e-7 relative over a full
    cycle plus a restart, and the explicit residual at the end matches."""
    if cplx:
        prob = P.helmholtz_shifted((16, 16, 14), omega2h2=1.0, damping=0.01)
    else:
        prob = P.laplacian_shifted((20, 20, 20), 0.6)
    prm = dict(levels=2, subdomains=8, rank=4, ilu="ilut")
    s, B, st, Pc = make_pair(prob, prm, tmp_path)
    b = P.rhs_vector(prob.n, cplx, 0)
    maxit = restart + 10
    out = s.solve(to_dev(s, b[st["perm"]]), rtol=1e-300, restart=restart, maxit=maxit)
    ref = oracle.fgmres(prob, b, M=Pc, rtol=1e-300, restart=restart, maxit=maxit)
    assert out["its"] == ref["its"] == maxit
    h = np.asarray(ref["hist"])
    assert h[restart] > 1e-6, "the problem converged too fast to exercise the late columns"
    assert np.allclose(out["hist"], h, rtol=1e-7, atol=0), np.abs(out["hist"] / h - 1).max()
    xg = np.empty(prob.n, dtype=b.dtype)
    xg[st["perm"]] = out["x"].cpu().numpy()
    assert rel(xg, ref["x"]) <= 1e-7
    assert out["final_relres"] == pytest.approx(ref["final_relres"], rel=1e-7)


@pytest.mark.parametrize("cplx,restart", [(False, 50), (False, 100), (True, 64), (True, 100)])
def test_dcgs2_every_column_count(tmp_path, cplx, restart):
    """DCGS2 (c5', reading Q38): one dot pass (column groups of 32) and one update pass
    per step at 1..restart columns, fp64 and complex, against the oracle's fgmres_dcgs2
    on the indefinite problems of the CGS2 test: same iteration count, histories equal to
    1e-7 relative over a full cycle plus a restart (the closing dot pass of every cycle
    completes its last column), the explicit residual and x."""
    if cplx:
        prob = P.helmholtz_shifted((16, 16, 14), omega2h2=1.0, damping=0.01)
    else:
        prob = P.laplacian_shifted((20, 20, 20), 0.6)
    prm = dict(levels=2, subdomains=8, rank=4, ilu="ilut")
    s, B, st, Pc = make_pair(prob, prm, tmp_path)
    b = P.rhs_vector(prob.n, cplx, 0)
    maxit = restart + 10
    out = s.solve(to_dev(s, b[st["perm"]]), rtol=1e-300, restart=restart, maxit=maxit, orth="dcgs2")
    ref = oracle.fgmres(prob, b, M=Pc, rtol=1e-300, restart=restart, maxit=maxit, orth="dcgs2")
    assert out["its"] == ref["its"] == maxit
    h = np.asarray(ref["hist"])
    assert len(out["hist"]) == len(h) == maxit + 1
    assert h[restart] > 1e-6, "the problem converged too fast to exercise the late columns"
    assert np.allclose(out["hist"], h, rtol=1e-7, atol=0), np.abs(out["hist"] / h - 1).max()
    xg = np.empty(prob.n, dtype=b.dtype)
    xg[st["perm"]] = out["x"].cpu().numpy()
    assert rel(xg, ref["x"]) <= 1e-7
    assert out["final_relres"] == pytest.approx(ref["final_relres"], rel=1e-7)
    # switching back on the same context: CGS2 graphs are captured again and agree with c5
    out2 = s.solve(to_dev(s, b[st["perm"]]), rtol=1e-300, restart=restart, maxit=12, orth="cgs2")
    ref2 = oracle.fgmres(prob, b, M=Pc, rtol=1e-300, restart=restart, maxit=12)
    assert np.allclose(out2["hist"], ref2["hist"], rtol=1e-7, atol=0)


@pytest.mark.parametrize("name,dims,over", CASES)
def test_dcgs2_solve_parity(tmp_path, name, dims, over):
    """Solves to the config tolerance with DCGS2 on both sides: iterations within +-1 of
    the oracle's fgmres_dcgs2, true residual <= rtol, histories while above the floor."""
    prob, b, xt, prm = P.make_config(name, dims=dims, **over)
    s, B, st, Pc = make_pair(prob, prm, tmp_path)
    perm = st["perm"]
    out = s.solve(to_dev(s, b[perm]), rtol=prm["rtol"], restart=prm["restart"], maxit=1000, orth="dcgs2")
    ref = oracle.fgmres(prob, b, M=Pc, rtol=prm["rtol"], restart=prm["restart"], maxit=1000, orth="dcgs2")
    assert out["status"] == 0 and ref["status"] == 0
    assert abs(out["its"] - ref["its"]) <= 1, (out["its"], ref["its"])
    xg = np.empty(prob.n, dtype=prob.values.dtype)
    xg[perm] = out["x"].cpu().numpy()
    true_rel = np.linalg.norm(b - oracle.spmv(prob, xg)) / np.linalg.norm(b)
    assert true_rel <= prm["rtol"]
    assert out["final_relres"] == pytest.approx(true_rel, rel=1e-6, abs=1e-14)
    h = min(len(out["hist"]), len(ref["hist"]))
    assert np.allclose(out["hist"][:h], ref["hist"][:h], rtol=1e-6, atol=1e2 * prm["rtol"])


@pytest.mark.slow
@pytest.mark.parametrize("name", ["C2", "C3", "C4", "C5"])
def test_full_size_parity(tmp_path, name):
    """BASELINE sizes (64^3 / 128^3; C5 is the configuration bench.py times): full-vector
    SpMV and apply parity, then the whole FGMRES solve on both sides — iterations within
    ±1 of the oracle and the true residual <= rtol (the north_star gate)."""
    prob, b, xt, prm = P.make_config(name)
    s, B, st, Pc = make_pair(prob, prm, tmp_path)
    perm = st["perm"]
    x = P.rhs_vector(prob.n, prob.is_complex, 13)
    y = s.spmv(to_dev(s, x[perm])).cpu().numpy()
    yo = oracle.spmv(prob, x)[perm]
    assert rel(y, yo) <= TOL
    yg = s.apply_precond(to_dev(s, x)).cpu().numpy()
    assert rel(yg, Pc.apply(x)) <= TOL
    out = s.solve(to_dev(s, b[perm]), rtol=prm["rtol"], restart=prm["restart"], maxit=1000)
    ref = oracle.fgmres(prob, b, M=Pc, rtol=prm["rtol"], restart=prm["restart"], maxit=1000)
    assert out["status"] == 0 and ref["status"] == 0
    assert abs(out["its"] - ref["its"]) <= 1, (out["its"], ref["its"])
    xg = np.empty(prob.n, dtype=b.dtype)
    xg[perm] = out["x"].cpu().numpy()
    true_rel = np.linalg.norm(b - oracle.spmv(prob, xg)) / np.linalg.norm(b)
    assert true_rel <= prm["rtol"], true_rel
    h = min(len(out["hist"]), len(ref["hist"]))
    assert np.allclose(out["hist"][:h], ref["hist"][:h], rtol=1e-6, atol=1e2 * prm["rtol"])
    # the same solve with DCGS2 (c5', the orthogonalisation bench.py times) on both sides
    out = s.solve(to_dev(s, b[perm]), rtol=prm["rtol"], restart=prm["restart"], maxit=1000, orth="dcgs2")
    ref = oracle.fgmres(prob, b, M=Pc, rtol=prm["rtol"], restart=prm["restart"], maxit=1000, orth="dcgs2")
    assert out["status"] == 0 and ref["status"] == 0
    assert abs(out["its"] - ref["its"]) <= 1, (out["its"], ref["its"])
    xg[perm] = out["x"].cpu().numpy()
    true_rel = np.linalg.norm(b - oracle.spmv(prob, xg)) / np.linalg.norm(b)
    assert true_rel <= prm["rtol"], true_rel


@pytest.mark.parametrize("name,dims,over", [("C5", (32, 32, 24), dict(subdomains=4, rank=4)),
                                             ("C4", (16, 16, 14), dict(subdomains=8, rank=6)),
                                             ("C3", (20, 18, 16), dict(subdomains=8, rank=0, ilu="ilu0")),
                                             ("C2", (24, 24, 24), dict(subdomains=4, rank=6, levels=3))])
@pytest.mark.parametrize("split", [2, 4])
def test_split_trisolve(tmp_path, name, dims, over, split):
    """The split form of the triangular solves (each subdomain's rows cut into 2 / 4
    contiguous chunks on the CTAs of a cluster, DSMEM hand-off of the values that cross
    chunks): apply parity (fp64 and c128, ILUT and ILU(0)), FGMRES iterations within ±1,
    and several right-hand sides at once."""
    prob, b, xt, prm = P.make_config(name, dims=dims, **over)
    s, B, st, Pc = make_pair(prob, prm, tmp_path, tri_split=split)
    stages = s.stats()["stages"]
    assert stages[0]["stage"]["split"] > 1, stages[0]
    for seed in (2, 3):
        r = P.rhs_vector(prob.n, prob.is_complex, seed)
        assert rel(s.apply_precond(to_dev(s, r)).cpu().numpy(), Pc.apply(r)) <= TOL
    out = s.solve(to_dev(s, b[st["perm"]]), rtol=prm["rtol"], restart=prm["restart"])
    ref = oracle.fgmres(prob, b, M=Pc, rtol=prm["rtol"], restart=prm["restart"])
    assert out["status"] == 0 and abs(out["its"] - ref["its"]) <= 1, (out["its"], ref["its"])
    cols = [P.rhs_vector(prob.n, prob.is_complex, 40 + c) for c in range(3)]
    X = torch.stack([to_dev(s, c) for c in cols])
    Y = s.apply_precond_multi(X).cpu().numpy()
    for c in range(3):
        assert rel(Y[c], Pc.apply(cols[c])) <= TOL


@pytest.mark.parametrize("kind", ["long_rows", "forced_stencil"])
def test_warp_per_row_spmv(tmp_path, kind, monkeypatch):
    """Warp-per-row CSR SpMV (k_spmv_wpr), chosen for long rows (>= 32 entries on average)
    or heavy SELL padding: SpMV and apply parity with the oracle, and an FGMRES solve."""
    import scipy.sparse as sp
    if kind == "long_rows":
        n = 3000
        M = sp.random(n, n, density=48.0 / n, random_state=7, format="csr")
        M = sp.csr_matrix(M + M.T + sp.identity(n) * 60.0)
        M.sort_indices()
        prob = P.Problem("long", (n,), M.indptr.astype(np.int64), M.indices.astype(np.int32), M.data, np.zeros((n, 3)))
        prm = dict(levels=2, subdomains=4, rank=4, ilu="ilut", ilut_drop=1e-3, ilut_fill=10)
        coords = False
    else:                                                          # the stencil with the kernel forced
        monkeypatch.setenv("GEMSLR_SPMV", "wpr")
        prob, b0, xt, prm = P.make_config("C3", dims=(20, 18, 16), subdomains=8, rank=6)
        coords = True
    s, B, st, Pc = make_pair(prob, prm, tmp_path, coords=coords)
    assert s.stats()["spmv_kernel"] == "wpr"
    perm = st["perm"]
    x = P.rhs_vector(prob.n, prob.is_complex, 4)
    y = s.spmv(to_dev(s, x[perm])).cpu().numpy()
    yn = np.empty_like(y)
    yn[perm] = y
    assert rel(yn, oracle.spmv(prob, x)) <= TOL
    assert rel(s.apply_precond(to_dev(s, x)).cpu().numpy(), Pc.apply(x)) <= TOL
    b = P.rhs_vector(prob.n, prob.is_complex, 9)
    out = s.solve(to_dev(s, b[perm]), rtol=1e-8, restart=30, maxit=500)
    ref = oracle.fgmres(prob, b, M=Pc, rtol=1e-8, restart=30, maxit=500)
    assert out["status"] == ref["status"] == 0 and abs(out["its"] - ref["its"]) <= 1


def _tail_suffix_ok(A, st):
    """Every level-l block's rows coupled to a later level (E_l's columns, F_l's rows)
    are its last rows (the order the tail sweeps rely on, DESIGN 6b)."""
    Ap = A[st["perm"]][:, st["perm"]].tocsr()
    Apt = Ap.T.tocsr()
    off = st["level_off"]
    for l, bl in enumerate(st["blocks"]):
        later = off[l + 1]
        for q in range(len(bl) - 1):
            a, e = int(bl[q]), int(bl[q + 1])
            coupled = [bool((Ap.indices[Ap.indptr[i]:Ap.indptr[i + 1]] >= later).any() or
                            (Apt.indices[Apt.indptr[i]:Apt.indptr[i + 1]] >= later).any()) for i in range(a, e)]
            if any(coupled):                  # exactly the coupled rows, after the others
                f = coupled.index(True)
                assert all(coupled[f:]), (l, q, f, sum(coupled[f:]), e - a - f)


@pytest.mark.parametrize("name,dims,over", [("C5", (32, 32, 24), dict(subdomains=4, rank=6)),
                                             ("C3", (24, 20, 20), dict(subdomains=8, rank=6)),
                                             ("C2", (24, 24, 24), dict(subdomains=4, rank=6, levels=3)),
                                             ("C5", (20, 20, 20), dict(subdomains=4, rank=0, ilu="ilu0"))])
def test_tail_form(tmp_path, monkeypatch, name, dims, over):
    """Boundary rows last in every B_l and the tail sweeps (DESIGN 6b): the coupled rows
    form a suffix of every block, every fp64 stage of levels 0..L-1 runs the tail form
    with shallower sweeps than the plain pair, and apply / solve parity hold with the
    oracle — with the tail form on and with it off (GEMSLR_TAIL=0, plain order)."""
    prob, b, xt, prm = P.make_config(name, dims=dims, **over)
    for tail in ("1", "0"):
        monkeypatch.setenv("GEMSLR_TAIL", tail)
        (tmp_path / f"t{tail}").mkdir()
        s, B, st, Pc = make_pair(prob, prm, tmp_path / f"t{tail}")
        stages = s.stats()["stages"]
        if tail == "1":
            _tail_suffix_ok(prob.scipy(), st)
            for g in stages:
                t = g["stage"]["tail"]
                assert t is not None, g["stage"]
                plain = g["stage"]["depth_L"] + g["stage"]["depth_U"]
                assert sum(t["depth_down"]) < plain and sum(t["depth_up"]) < plain + 8, (t, plain)
        else:
            assert all(g["stage"]["tail"] is None for g in stages)
        for seed in (2, 3):
            r = P.rhs_vector(prob.n, prob.is_complex, seed)
            assert rel(s.apply_precond(to_dev(s, r)).cpu().numpy(), Pc.apply(r)) <= TOL
        for orth in ("cgs2", "dcgs2"):              # DCGS2: pre-packed level 0 in the tail form only
            out = s.solve(to_dev(s, b[st["perm"]]), rtol=prm["rtol"], restart=prm["restart"], orth=orth)
            ref = oracle.fgmres(prob, b, M=Pc, rtol=prm["rtol"], restart=prm["restart"], orth=orth)
            assert out["status"] == 0 and abs(out["its"] - ref["its"]) <= 1, (orth, out["its"], ref["its"])
            xg = np.empty(prob.n)
            xg[st["perm"]] = out["x"].cpu().numpy()
            assert np.linalg.norm(b - oracle.spmv(prob, xg)) <= prm["rtol"] * np.linalg.norm(b)
        s.close()
