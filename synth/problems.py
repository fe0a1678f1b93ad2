"""Seeded synthetic inputs shared by the oracle tests, the GPU tests and bench.py.

This module holds NO arithmetic of the method (no preconditioner, no Krylov
step).  It only writes down the test matrices of the BASELINE configs and
draws their right-hand sides, as fixed by SURVEY.md §8(c) c1 and DESIGN.md
"Input recipe":

* grids hold interior points only (homogeneous Dirichlet values eliminated),
  lexicographic index i = x + Nx*(y + Ny*z), x fastest, h = 1/(N+1)
  (model problem, eq. test_problem_1);
* stencils are h^2-scaled (reading Q17): 5-pt diag 4 / 7-pt diag 6, -1 per
  existing neighbour; upwind convection-diffusion (Q18); complex shifted
  Helmholtz (Q19);
* right-hand sides from numpy.random.default_rng(seed) (Q20): real
  v = uniform(-1,1,N); complex re then im.  For the "manufactured" configs
  (C2, C5) x_true = v and b = A @ x_true, computed with scipy's CSR product
  (a library primitive generating the problem, not a step of the method).

Matrices are returned as (rowptr int64, colidx int32, values float64 or
complex128) CSR with sorted unique columns, plus integer grid coordinates
(used by the product's optional coordinate bisection).
"""
from __future__ import annotations

import dataclasses
import numpy as np


@dataclasses.dataclass
class Problem:
    name: str
    dims: tuple
    rowptr: np.ndarray   # int64 [n+1]
    colidx: np.ndarray   # int32 [nnz]
    values: np.ndarray   # float64 or complex128 [nnz]
    coords: np.ndarray   # float64 [n, 3] grid coordinates (x, y, z)

    @property
    def n(self) -> int:
        return len(self.rowptr) - 1

    @property
    def nnz(self) -> int:
        return int(self.rowptr[-1])

    @property
    def is_complex(self) -> bool:
        return np.iscomplexobj(self.values)

    def scipy(self):
        import scipy.sparse as sp
        return sp.csr_matrix((self.values, self.colidx.astype(np.int64), self.rowptr),
                             shape=(self.n, self.n))


def _stencil(dims, diag, lower, upper, dtype=np.float64, name="stencil"):
    """Generic 2D/3D structured stencil.

    dims = (Nx, Ny[, Nz]); `lower[a]` is the coefficient of the neighbour at
    coordinate -1 along axis a, `upper[a]` the one at +1.  Columns come out in
    ascending order because the neighbours are emitted in index order
    (z-1, y-1, x-1, self, x+1, y+1, z+1).
    """
    dims = tuple(int(d) for d in dims)
    nd = len(dims)
    n = int(np.prod(dims))
    idx = np.arange(n, dtype=np.int64)
    crd = []
    rem = idx.copy()
    for d in dims:
        crd.append(rem % d)
        rem //= d
    strides = [1]
    for d in dims[:-1]:
        strides.append(strides[-1] * d)
    # emission order: descending axes for "lower", then self, then ascending axes for "upper"
    entries = []  # (mask, col, value)
    for a in reversed(range(nd)):
        m = crd[a] > 0
        entries.append((m, idx - strides[a], lower[a]))
    entries.append((np.ones(n, dtype=bool), idx, diag))
    for a in range(nd):
        m = crd[a] < dims[a] - 1
        entries.append((m, idx + strides[a], upper[a]))
    counts = np.zeros(n, dtype=np.int64)
    for m, _, _ in entries:
        counts += m
    rowptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(counts, out=rowptr[1:])
    nnz = int(rowptr[-1])
    colidx = np.empty(nnz, dtype=np.int32)
    values = np.empty(nnz, dtype=dtype)
    pos = rowptr[:-1].copy()
    for m, col, val in entries:
        where = pos[m]
        colidx[where] = col[m]
        values[where] = val
        pos[m] += 1
    coords = np.zeros((n, 3), dtype=np.float64)
    for a in range(nd):
        coords[:, a] = crd[a]
    return Problem(name, dims, rowptr, colidx, values, coords)


def laplacian(dims, name=None):
    """5-pt (2D) or 7-pt (3D) negative Laplacian, h^2-scaled: diag 2d, -1 per neighbour."""
    nd = len(dims)
    return _stencil(dims, 2.0 * nd, [-1.0] * nd, [-1.0] * nd,
                    name=name or f"laplacian{nd}d_{'x'.join(map(str, dims))}")


def convdiff_upwind(dims, beta=(20.0, 20.0, 20.0), name=None):
    """-Δu + β·∇u, first-order upwind for β > 0 (reading Q18), h^2-scaled.

    diag = 2d + h Σβ_a; upstream neighbour (coordinate -1) -1 - h β_a;
    downstream -1.  h = 1/(N+1) of axis 0 (cubes in the configs).
    """
    nd = len(dims)
    h = 1.0 / (dims[0] + 1)
    diag = 2.0 * nd + h * float(sum(beta[:nd]))
    lower = [-1.0 - h * beta[a] for a in range(nd)]
    upper = [-1.0] * nd
    return _stencil(dims, diag, lower, upper,
                    name=name or f"convdiff{nd}d_{'x'.join(map(str, dims))}")


def helmholtz_shifted(dims, omega2h2=0.1, damping=0.5, name=None):
    """-Δu - (ω² + damping·iω²)u, h^2-scaled: diag 2d - ω²h²(1 + damping·i) (reading Q19;
    C4 is ω²h² = 0.1, damping 0.5), c128."""
    nd = len(dims)
    diag = complex(2.0 * nd - omega2h2, -damping * omega2h2)
    return _stencil(dims, diag, [-1.0 + 0j] * nd, [-1.0 + 0j] * nd, dtype=np.complex128,
                    name=name or f"helmholtz{nd}d_{'x'.join(map(str, dims))}")


def laplacian_shifted(dims, sigma, name=None):
    """The 7-pt / 5-pt Laplacian with diagonal 2d - sigma: indefinite for sigma above its
    smallest eigenvalue (a real analogue of the Helmholtz operator; test input only)."""
    nd = len(dims)
    return _stencil(dims, 2.0 * nd - sigma, [-1.0] * nd, [-1.0] * nd,
                    name=name or f"laplacian_shift{sigma}_{'x'.join(map(str, dims))}")


def rhs_vector(n, is_complex, seed=0):
    """Q20: numpy.random.default_rng(seed); real uniform(-1,1); complex re then im."""
    rng = np.random.default_rng(seed)
    if is_complex:
        re = rng.uniform(-1.0, 1.0, n)
        im = rng.uniform(-1.0, 1.0, n)
        return re + 1j * im
    return rng.uniform(-1.0, 1.0, n)


def manufactured_rhs(prob: Problem, seed=0):
    """x_true = uniform(-1,1) from the seed, b = A x_true (C2/C5)."""
    x_true = rhs_vector(prob.n, prob.is_complex, seed)
    b = prob.scipy() @ x_true
    return b, x_true


# ---------------------------------------------------------------------------
# BASELINE.json configs C1-C5.  `levels`, `subdomains`,
# `rank` are the parameters of setup(A, levels, k=p, rank) (reading Q31).
# ---------------------------------------------------------------------------
CONFIGS = {
    "C1": dict(kind="laplacian", dims=(32, 32), levels=1, subdomains=4, rank=8,
               ilu="ilu0", restart=30, rtol=1e-8, rhs="uniform"),
    "C2": dict(kind="laplacian", dims=(64, 64, 64), levels=2, subdomains=16, rank=20,
               ilu="ilut", restart=50, rtol=1e-8, rhs="manufactured"),
    "C3": dict(kind="convdiff", dims=(128, 128, 128), levels=3, subdomains=64, rank=32,
               ilu="ilut", restart=50, rtol=1e-6, rhs="uniform"),
    "C4": dict(kind="helmholtz", dims=(128, 128, 128), levels=3, subdomains=64, rank=40,
               ilu="ilut", restart=100, rtol=1e-6, rhs="uniform"),
    "C5": dict(kind="laplacian", dims=(128, 128, 128), levels=3, subdomains=32, rank=20,
               ilu="ilut", restart=50, rtol=1e-8, rhs="manufactured"),
}

ILUT_DROP = 1e-3   # BASELINE C2 "ILUT(drop 1e-3, fill 10)"; Q9/Q10
ILUT_FILL = 10


def c5_dims(gpus: int):
    """Weak-scaling grid of C5: 128^3 per GPU (G=2: 256x128x128, G=4: 256x256x128, G=8: 256^3)."""
    return {1: (128, 128, 128), 2: (256, 128, 128), 4: (256, 256, 128),
            8: (256, 256, 256)}[gpus]


def make_matrix(kind, dims, **kw):
    if kind == "laplacian":
        return laplacian(dims)
    if kind == "convdiff":
        return convdiff_upwind(dims)
    if kind == "helmholtz":
        return helmholtz_shifted(dims, **kw)
    raise ValueError(kind)


def make_config(name, dims=None, seed=0, gpus=1, **overrides):
    """Return (Problem, b, x_true_or_None, params) for config `name`.

    `dims` overrides the grid (used by tests to run the same recipe small).
    """
    cfg = dict(CONFIGS[name])
    cfg.update(overrides)
    if dims is None:
        dims = c5_dims(gpus) if name == "C5" else cfg["dims"]
        if name == "C5":
            cfg["subdomains"] = 32 * gpus
    prob = make_matrix(cfg["kind"], dims, **{k: cfg[k] for k in ("omega2h2", "damping") if k in cfg})
    prob.name = f"{name}:{prob.name}"
    if cfg["rhs"] == "manufactured":
        b, x_true = manufactured_rhs(prob, seed)
    else:
        b, x_true = rhs_vector(prob.n, prob.is_complex, seed), None
    params = dict(levels=cfg["levels"], subdomains=cfg["subdomains"], rank=cfg["rank"],
                  ilu=cfg["ilu"], ilut_drop=ILUT_DROP, ilut_fill=ILUT_FILL,
                  restart=cfg["restart"], rtol=cfg["rtol"])
    return prob, b, x_true, params


def expected_nnz(dims):
    """Closed form (2d+1)·N − 2·Σ_axes N/N_axis."""
    n = int(np.prod(dims))
    return (2 * len(dims) + 1) * n - 2 * sum(n // d for d in dims)
