"""Pins of the seeded input generators (SURVEY.md §8(c) c8 "Generators")."""
import numpy as np
import pytest

from synth import problems as P


@pytest.mark.parametrize("dims,expect", [((32, 32), 4992), ((64, 64, 64), 1810432), ((5, 7, 3), None)])
def test_nnz_closed_form(dims, expect):
    A = P.laplacian(dims)
    assert A.nnz == P.expected_nnz(dims)
    if expect is not None:
        assert A.nnz == expect          # SURVEY.md §8(a) table (4,992 / 1,810,432)


def test_nnz_128_closed_form_value():
    # 14,581,760 and 117,047,296 (C3-C5, C5 at G=8) from the closed form alone
    assert P.expected_nnz((128, 128, 128)) == 14581760
    assert P.expected_nnz((256, 256, 256)) == 117047296


@pytest.mark.parametrize("dims", [(6, 5), (4, 5, 6)])
def test_laplacian_symmetric_and_row_sums(dims):
    A = P.laplacian(dims).scipy()
    assert abs(A - A.T).max() == 0.0
    # (A·1)_i = number of Dirichlet faces of point i (exact integers)
    crd = np.array(np.unravel_index(np.arange(A.shape[0]), dims[::-1])[::-1]).T
    faces = np.zeros(A.shape[0])
    for a, d in enumerate(dims):
        faces += (crd[:, a] == 0) + (crd[:, a] == d - 1)
    assert np.array_equal(A @ np.ones(A.shape[0]), faces)


def test_columns_sorted_unique_and_diag():
    for prob in (P.laplacian((7, 6, 5)), P.convdiff_upwind((7, 6, 5)), P.helmholtz_shifted((4, 4, 4))):
        for i in range(prob.n):
            c = prob.colidx[prob.rowptr[i]:prob.rowptr[i + 1]]
            assert np.all(np.diff(c) > 0)
            assert i in c


def test_convdiff_stencil_values():
    n = 9
    A = P.convdiff_upwind((n, n, n)).scipy()
    h = 1.0 / (n + 1)
    i = 4 + n * (4 + n * 4)   # interior point
    assert A[i, i] == pytest.approx(6 + 60 * h, rel=0, abs=1e-15)
    for s in (1, n, n * n):
        assert A[i, i - s] == pytest.approx(-1 - 20 * h, abs=1e-15)   # upstream (Q18)
        assert A[i, i + s] == -1.0
    # interior row sums vanish: 6 + 60h - 3(1 + 20h) - 3 = 0
    assert abs((A @ np.ones(A.shape[0]))[i]) < 1e-14
    assert abs(A - A.T).max() > 0       # nonsymmetric


def test_helmholtz_diag():
    A = P.helmholtz_shifted((4, 4, 4)).scipy()
    assert A[0, 0] == complex(5.9, -0.05)      # 6 - 0.1(1 + 0.5i), Q19
    assert A.dtype == np.complex128


def test_rhs_seeded():
    a = P.rhs_vector(100, False, 0)
    b = P.rhs_vector(100, False, 0)
    assert np.array_equal(a, b) and a.min() >= -1 and a.max() <= 1
    z = P.rhs_vector(100, True, 0)
    assert np.array_equal(z.real, np.random.default_rng(0).uniform(-1, 1, 100))


def test_config_shapes():
    prob, b, xt, prm = P.make_config("C1")
    assert prob.n == 1024 and prob.nnz == 4992 and xt is None and prm["rank"] == 8
    prob, b, xt, prm = P.make_config("C2", dims=(8, 8, 8))
    assert xt is not None and np.allclose(prob.scipy() @ xt, b)
