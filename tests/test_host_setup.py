"""CPU tests of the product's host stage (host-only context, device = -1) and
of the C-ABI surface, verified by the independent oracle.
No GPU compute is called here."""
import os
import re

import numpy as np
import pytest
import scipy.sparse as sp

import oracle
from oracle import dense as D
from synth import problems as P
from tests.bundle_io import Bundle

gm = pytest.importorskip("paper_2205_03224_b200")


@pytest.fixture(scope="module", autouse=True)
def built():
    from paper_2205_03224_b200 import build
    build.build()


def test_library_exports_every_header_symbol():
    hdr = open(os.path.join(os.path.dirname(__file__), "..", "include", "gemslr.h")).read()
    names = set(re.findall(r"^(?:gemslr_status|const char\s*\*|void)\s*\*?\s*(gemslr_\w+)\s*\(", hdr, re.M))
    assert names == set(gm.ABI_FUNCTIONS)
    L = gm.lib()
    for nm in names:
        assert hasattr(L, nm), nm


def host_solver(prob, levels, p, ilu="ilut", coords=True, **kw):
    return gm.Solver(prob.rowptr, prob.colidx, prob.values, levels, p, 0, ilu=ilu,
                     coords=prob.coords if coords else None, device=-1, **kw)


def verify_bundle_host(prob, s, tmp_path, ilu_kind, tau, lfil):
    d = s.export(str(tmp_path / "bundle"))
    B = Bundle(d)
    st = B.structure()
    n = prob.n
    assert D.verify_perm(st["perm"], n)                          # c3.1
    A = prob.scipy()
    Ah = D.permute_matrix(A, st["perm"])                          # oracle's own Â
    assert D.verify_separators(Ah, st["level_off"], st["blocks"]) == 0   # c3.2
    o = st["level_off"]
    assert o[0] == 0 and np.all(np.diff(o) >= 0)
    for l, bl in enumerate(st["blocks"]):
        assert bl[0] == o[l] and bl[-1] == o[l + 1] and np.all(np.diff(bl) >= 0)
    assert st["last_off"][0] == o[-1] and st["last_off"][-1] == n
    # factors: the oracle recomputes every block from its own Â and compares (c3.3/c3.4)
    Pc = oracle.Precond(A, st, ilu=(ilu_kind, tau, lfil))
    mism = 0
    worst = 0.0
    L = len(o) - 1
    for l in range(L + 1):
        tag = "faclast" if l == L else f"fac{l}"
        for which, wi in (("L", 0), ("U", 1)):
            for q, Fb in enumerate(B.factors(tag, which)):
                Fo = Pc.factor(l, q, wi)
                if not D.pattern_equal(Fb, Fo):
                    mism += 1
                    continue
                if Fb.nnz:
                    worst = max(worst, np.abs(Fb.data - Fo.data).max() / np.abs(Fo.data).max())
    assert mism == 0
    assert worst <= 1e-12
    if ilu_kind == oracle.ILU0:                                   # defining property on every block
        bl = st["blocks"][0]
        Lf, Uf = B.factors("fac0", "L"), B.factors("fac0", "U")
        for q in range(len(bl) - 1):
            Bq = Ah[bl[q]:bl[q + 1], bl[q]:bl[q + 1]]
            if Bq.shape[0]:
                assert D.ilu0_property_error(Bq, Lf[q], Uf[q]) < 1e-13
    return B, st


@pytest.mark.parametrize("ilu", ["ilu0", "ilut"])
def test_host_plan_C1_recipe(tmp_path, ilu):
    prob, b, _, prm = P.make_config("C1")
    s = host_solver(prob, prm["levels"], prm["subdomains"], ilu=ilu)
    kind = oracle.ILU0 if ilu == "ilu0" else oracle.ILUT
    B, st = verify_bundle_host(prob, s, tmp_path, kind, 1e-3, 10)
    assert B.L == 1 and len(st["blocks"][0]) == 5


@pytest.mark.parametrize("make,levels,p,coords", [
    (lambda: P.laplacian((12, 12, 12)), 3, 8, True),
    (lambda: P.convdiff_upwind((10, 9, 8)), 2, 4, True),
    (lambda: P.helmholtz_shifted((8, 8, 8)), 3, 4, True),
    (lambda: P.laplacian((16, 16)), 2, 4, False),          # BFS bisection (no coordinates)
])
def test_host_plan_multilevel(tmp_path, make, levels, p, coords):
    prob = make()
    s = host_solver(prob, levels, p, coords=coords, ilut_drop=1e-3, ilut_fill=10)
    B, st = verify_bundle_host(prob, s, tmp_path, oracle.ILUT, 1e-3, 10)
    stats = s.stats()
    assert stats["levels"] == B.L >= 1
    assert stats["fill"] > 1.0


def test_rcb_on_cube_gives_face_line_point_hierarchy():
    prob = P.laplacian((32, 32, 32))
    s = host_solver(prob, 3, 8)
    o = s.stats()["level_off"]
    sizes = np.diff(o + [prob.n])
    # level-0 separator = faces (~3 planes of 32^2), level-1 = lines, last = points
    assert sizes[0] > 0.85 * prob.n
    assert 2000 < prob.n - o[1] < 4000
    assert prob.n - o[-1] < 200


def test_errors_are_reported():
    prob = P.laplacian((4, 4))
    with pytest.raises(gm.GemslrError) as e:
        gm.Solver(prob.rowptr, prob.colidx, prob.values, 1, 100, 0, device=-1)
    assert e.value.code == -3                                 # PARTITION
    bad = prob.colidx.copy()
    bad[1], bad[2] = bad[2], bad[1]
    with pytest.raises(gm.GemslrError) as e:
        gm.Solver(prob.rowptr, bad, prob.values, 1, 2, 0, device=-1)
    assert e.value.code == -2                                 # BAD_CSR
    with pytest.raises(gm.GemslrError) as e:
        gm.Solver(prob.rowptr, prob.colidx, prob.values, 0, 2, 0, device=-1)
    assert e.value.code == -1                                 # INVALID_ARG
    z = prob.values.copy()
    z[prob.rowptr[0]:prob.rowptr[1]] = 0.0                    # zero row -> zero pivot
    with pytest.raises(gm.GemslrError) as e:
        gm.Solver(prob.rowptr, prob.colidx, z, 1, 2, 0, ilu="ilu0", device=-1)
    assert e.value.code == -4 and "row" in str(e.value)


def test_host_only_context_refuses_device_calls():
    prob = P.laplacian((6, 6))
    s = host_solver(prob, 1, 2)
    rc = gm.lib().gemslr_apply_precond(s.h, None, None)
    assert rc in (-1, -6)


def test_orthogonalization_setter():
    """gemslr_set_orthogonalization: 0 (CGS2) and 1 (DCGS2, reading Q38) accepted on any
    context, anything else INVALID_ARG; the binding maps the names and rejects others."""
    prob = P.laplacian((6, 6))
    s = host_solver(prob, 1, 2)
    assert gm.lib().gemslr_set_orthogonalization(s.h, 0) == 0
    assert gm.lib().gemslr_set_orthogonalization(s.h, 1) == 0
    assert gm.lib().gemslr_set_orthogonalization(s.h, 2) == -1
    assert gm.lib().gemslr_set_orthogonalization(s.h, -1) == -1
    assert gm.lib().gemslr_set_orthogonalization(None, 1) == -1
    s.set_orthogonalization("dcgs2")
    assert s.orth == "dcgs2"
    with pytest.raises(ValueError):
        s.set_orthogonalization("mgs")
