"""Pins against values the paper prints (tests/golden/, each fixture cites its passage)."""
import os

import numpy as np

from synth import problems as P

HERE = os.path.dirname(os.path.abspath(__file__))


def _fixture(name):
    d = {}
    for line in open(os.path.join(HERE, "golden", name)):
        line = line.strip()
        if line and not line.startswith("#"):
            k, v = line.split()
            d[k] = float(v)
    return d


def test_shifted_laplacian_spectrum_P_L1392():
    """the shifted 30 x 20 Laplacian (n = 600, shift 1.0) has its spectrum nearly
    evenly distributed in [-1, 7] — checked on the generator's 5-point Laplacian."""
    g = _fixture("shifted_laplacian_30x20.txt")
    prob = P.laplacian((int(g["nx"]), int(g["ny"])))
    assert prob.n == int(g["n"])
    A = np.zeros((prob.n, prob.n))
    for i in range(prob.n):
        for p in range(prob.rowptr[i], prob.rowptr[i + 1]):
            A[i, prob.colidx[p]] = prob.values[p]
    assert np.allclose(A, A.T)
    ev = np.linalg.eigvalsh(A - g["shift"] * np.eye(prob.n))
    lo, hi = g["spectrum_lo"], g["spectrum_hi"]
    assert lo < ev.min() < lo + 0.05 and hi - 0.05 < ev.max() < hi
    # "nearly evenly": every eighth of the interval holds between 0.6x and 1.6x of its share
    # (measured 46 ... 117 of 75; the 2D density peaks at the centre, symmetric about 3)
    counts, _ = np.histogram(ev, bins=8, range=(lo, hi))
    share = prob.n / 8
    assert counts.min() >= 0.6 * share and counts.max() <= 1.6 * share, counts
    assert np.array_equal(counts, counts[::-1])
