"""ORACLE — test infrastructure only (see oracle/oracle.cpp header).

Thin ctypes/numpy wrapper over the plain C++ oracle (liboracle.so) plus a few
plain NumPy/SciPy helpers.  Only tests/, __graft_entry__.smoke() and
bench.py (cpu_baseline and --impl reference) may import this package; the
product package never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
_SRC = os.path.join(_HERE, "oracle.cpp")

_lib = None


def build(force=False):
    """Compile liboracle.so (g++ -O2 -ffp-contract=off -fopenmp; reading Q22; thread-count
    independent results, oracle.cpp header)."""
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(_SRC):
        cmd = ["g++", "-std=c++17", "-O2", "-ffp-contract=off", "-fopenmp", "-fPIC", "-shared",
               "-o", _SO + ".tmp", _SRC]
        subprocess.check_call(cmd)
        os.replace(_SO + ".tmp", _SO)
    return _SO


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(_SO)
        vp, i64, i32p, i64p, dp = C.c_void_p, C.c_int64, C.POINTER(C.c_int32), C.POINTER(C.c_int64), C.POINTER(C.c_double)
        L.or_spmv.argtypes = [C.c_int, i64, vp, vp, vp, vp, vp]
        L.or_set_threads.argtypes = [C.c_int]
        L.or_get_threads.restype = C.c_int
        L.or_ilu_create.argtypes = [C.c_int, i64, vp, vp, vp, C.c_int, C.c_double, C.c_int, C.c_char_p, C.c_int]
        L.or_ilu_create.restype = vp
        L.or_ilu_nnz.argtypes = [vp, C.c_int]
        L.or_ilu_nnz.restype = i64
        L.or_ilu_get.argtypes = [vp, C.c_int, vp, vp, vp]
        L.or_ilu_solve.argtypes = [vp, vp, vp]
        L.or_ilu_destroy.argtypes = [vp]
        L.or_precond_create.argtypes = [C.c_int, i64, vp, vp, vp, vp, C.c_int, vp, vp, vp, C.c_int, vp,
                                        C.c_int, C.c_double, C.c_int, C.c_double, C.c_char_p, C.c_int]
        L.or_precond_create.restype = vp
        L.or_precond_destroy.argtypes = [vp]
        L.or_precond_set_root_its.argtypes = [vp, C.c_int]
        L.or_precond_set_lowrank.argtypes = [vp, C.c_int, C.c_int, vp, vp]
        L.or_precond_apply_from.argtypes = [vp, C.c_int, vp, vp]
        L.or_ghat.argtypes = [vp, C.c_int, vp, vp]
        L.or_precond_natural.argtypes = [vp, vp, vp]
        L.or_precond_factor_nnz.argtypes = [vp, C.c_int, C.c_int, C.c_int]
        L.or_precond_factor_nnz.restype = i64
        L.or_precond_factor_get.argtypes = [vp, C.c_int, C.c_int, C.c_int, vp, vp, vp]
        L.or_fgmres.argtypes = [C.c_int, i64, vp, vp, vp, vp, vp, vp, vp, C.c_double, C.c_int, C.c_int,
                                C.POINTER(C.c_int), dp, C.c_int, C.POINTER(C.c_int), dp, C.c_int, dp]
        L.or_fgmres.restype = C.c_int
        L.or_fgmres_dcgs2.argtypes = L.or_fgmres.argtypes
        L.or_fgmres_dcgs2.restype = C.c_int
        _lib = L
    return _lib


def set_threads(n):
    """OpenMP threads of the oracle (results are the same for any count)."""
    lib().or_set_threads(int(n))


def get_threads():
    return int(lib().or_get_threads())


def _p(a):
    return a.ctypes.data_as(C.c_void_p)


def _csr_args(rowptr, colidx, values):
    rowptr = np.ascontiguousarray(rowptr, dtype=np.int64)
    colidx = np.ascontiguousarray(colidx, dtype=np.int32)
    cplx = np.iscomplexobj(values)
    values = np.ascontiguousarray(values, dtype=np.complex128 if cplx else np.float64)
    return rowptr, colidx, values, int(cplx)


def as_csr(A):
    """(rowptr, colidx, values) from a synth Problem or a scipy matrix."""
    if hasattr(A, "rowptr"):
        return A.rowptr, A.colidx, A.values
    A = A.tocsr()
    A.sort_indices()
    return A.indptr.astype(np.int64), A.indices.astype(np.int32), A.data


def spmv(A, x):
    """c2: y = A x, y_i = Σ_j a_ij x_j (j ascending), natural order."""
    rp, ci, v, cplx = _csr_args(*as_csr(A))
    x = np.ascontiguousarray(x, dtype=v.dtype)
    y = np.empty(len(rp) - 1, dtype=v.dtype)
    lib().or_spmv(cplx, len(rp) - 1, _p(rp), _p(ci), _p(v), _p(x), _p(y))
    return y


ILU0, ILUT = 0, 1


class Ilu:
    """ILU(0) / ILUT(τ, lfil) of one matrix (oracle.cpp ilu0 / ilut)."""

    def __init__(self, A, kind=ILU0, tau=0.0, lfil=1 << 30):
        rp, ci, v, cplx = _csr_args(*as_csr(A))
        self.n = len(rp) - 1
        self.dtype = v.dtype
        err = C.create_string_buffer(512)
        self.h = lib().or_ilu_create(cplx, self.n, _p(rp), _p(ci), _p(v), kind, tau, int(min(lfil, 2**31 - 1)), err, 512)
        if not self.h:
            raise RuntimeError(err.value.decode())

    def factor(self, which):
        import scipy.sparse as sp
        nnz = lib().or_ilu_nnz(self.h, which)
        ptr = np.empty(self.n + 1, np.int64)
        col = np.empty(nnz, np.int64)
        val = np.empty(nnz, self.dtype)
        lib().or_ilu_get(self.h, which, _p(ptr), _p(col), _p(val))
        return sp.csr_matrix((val, col, ptr), shape=(self.n, self.n))

    @property
    def L(self):
        return self.factor(0)

    @property
    def U(self):
        return self.factor(1)

    def solve(self, b):
        b = np.ascontiguousarray(b, dtype=self.dtype)
        x = np.empty_like(b)
        lib().or_ilu_solve(self.h, _p(b), _p(x))
        return x

    def __del__(self):
        try:
            if getattr(self, "h", None):
                lib().or_ilu_destroy(self.h)
                self.h = None
        except Exception:                                          # interpreter shutdown
            pass


class Precond:
    """The GeMSLR preconditioner (Alg. 2, c4) on a given multilevel structure.

    structure: dict with
      perm        int64 [N]  perm[new] = old
      level_off   int64 [L+1] o_0..o_L (o_L = start of C_last)
      blocks      list of L int64 arrays of absolute block boundaries per level
      last_off    int64 array of absolute C_last block boundaries
    ilu: (kind, tau, lfil).  Factors are computed by the oracle itself.
    shift: complex diagonal shift factor of the block ILUs, sigma = i*shift*sum|a_ii|/n
    (reading Q33; complex problems only).
    """

    def __init__(self, A, structure, ilu=(ILU0, 0.0, 0), shift=0.0):
        rp, ci, v, cplx = _csr_args(*as_csr(A))
        self.n = len(rp) - 1
        self.dtype = v.dtype
        self.cplx = cplx
        self.perm = np.ascontiguousarray(structure["perm"], dtype=np.int64)
        self.o = np.ascontiguousarray(structure["level_off"], dtype=np.int64)
        self.L = len(self.o) - 1
        blocks = [np.asarray(b, dtype=np.int64) for b in structure["blocks"]]
        nblk = np.array([len(b) - 1 for b in blocks], dtype=np.int32)
        blk_off = np.ascontiguousarray(np.concatenate(blocks) if blocks else np.zeros(0, np.int64), dtype=np.int64)
        last = np.ascontiguousarray(structure["last_off"], dtype=np.int64)
        self.last_off = last
        self.blocks = blocks
        err = C.create_string_buffer(1024)
        kind, tau, lfil = ilu
        self.h = lib().or_precond_create(cplx, self.n, _p(rp), _p(ci), _p(v), _p(self.perm), self.L, _p(self.o),
                                         _p(nblk), _p(blk_off), len(last) - 1, _p(last), int(kind), float(tau),
                                         int(min(lfil, 2**31 - 1)), float(shift), err, 1024)
        if not self.h:
            raise RuntimeError(err.value.decode())
        self._keep = (rp, ci, v)

    def s(self, l):
        return int(self.n - self.o[l + 1])

    def set_root_its(self, its):
        """NEXT-1: `its` steps of right-preconditioned GMRES on Ŝ_0 at the root level (0 = single pass)."""
        lib().or_precond_set_root_its(self.h, int(its))

    def set_lowrank(self, l, W, G):
        W = np.asfortranarray(W, dtype=self.dtype)
        G = np.asfortranarray(G, dtype=self.dtype)
        k = W.shape[1] if W.ndim == 2 else 0
        assert W.shape[0] == self.s(l)
        lib().or_precond_set_lowrank(self.h, l, k, _p(W), _p(G))

    def apply(self, r, l0=0):
        """y = M^{-1} r in the permuted order (l0 > 0: C_{l0-1}^{-1} on [o_l0, N))."""
        r = np.ascontiguousarray(r, dtype=self.dtype)
        y = np.empty_like(r)
        lib().or_precond_apply_from(self.h, l0, _p(r), _p(y))
        return y

    def apply_natural(self, x):
        x = np.ascontiguousarray(x, dtype=self.dtype)
        y = np.empty_like(x)
        lib().or_precond_natural(self.h, _p(x), _p(y))
        return y

    def ghat(self, l, v):
        v = np.ascontiguousarray(v, dtype=self.dtype)
        out = np.empty(self.s(l), dtype=self.dtype)
        lib().or_ghat(self.h, l, _p(v), _p(out))
        return out

    def factor(self, l, q, which):
        """(L or U) factor of block q of level l (l == L: C_last block q) as scipy CSR."""
        import scipy.sparse as sp
        nnz = lib().or_precond_factor_nnz(self.h, l, q, which)
        if l == self.L:
            nb = int(self.last_off[q + 1] - self.last_off[q])
        else:
            nb = int(self.blocks[l][q + 1] - self.blocks[l][q])
        ptr = np.empty(nb + 1, np.int64)
        col = np.empty(nnz, np.int64)
        val = np.empty(nnz, self.dtype)
        lib().or_precond_factor_get(self.h, l, q, which, _p(ptr), _p(col), _p(val))
        return sp.csr_matrix((val, col, ptr), shape=(nb, nb))

    def natural_fn(self):
        """(function pointer, user pointer) usable by fgmres as M_nat^{-1} = P M^{-1} Pᵀ."""
        return C.cast(lib().or_precond_natural, C.c_void_p), C.c_void_p(self.h)

    def __del__(self):
        try:
            if getattr(self, "h", None):
                lib().or_precond_destroy(self.h)
                self.h = None
        except Exception:                                          # interpreter shutdown
            pass


_PRECOND_FN = C.CFUNCTYPE(None, C.c_void_p, C.c_void_p, C.c_void_p)


def fgmres(A, b, x0=None, M=None, rtol=1e-8, restart=30, maxit=1000, diag=False, orth="cgs2"):
    """c5: FGMRES(m) with CGS2 on natural-order A (orth="dcgs2": c5', the lagged
    DCGS2 variant of reading Q38).

    M: None (identity), an oracle.Precond (applied as P M^{-1} Pᵀ), or a
    Python callable v -> z (e.g. a dense solve in the pins).
    Returns dict(x, its, hist, final_relres, status[, orth, arnoldi, est_gap]).
    """
    rp, ci, v, cplx = _csr_args(*as_csr(A))
    n = len(rp) - 1
    b = np.ascontiguousarray(b, dtype=v.dtype)
    x = np.zeros(n, dtype=v.dtype) if x0 is None else np.array(x0, dtype=v.dtype)
    keep = None
    if M is None:
        fn, user = None, None
    elif isinstance(M, Precond):
        fn, user = M.natural_fn()
    else:
        dt = v.dtype

        def cb(_user, pin, pout):
            vin = np.ctypeslib.as_array(C.cast(pin, C.POINTER(C.c_double)), shape=(n * (2 if cplx else 1),))
            vout = np.ctypeslib.as_array(C.cast(pout, C.POINTER(C.c_double)), shape=(n * (2 if cplx else 1),))
            z = np.asarray(M(vin.view(dt).copy()), dtype=dt)
            vout[:] = z.view(np.float64)
        keep = _PRECOND_FN(cb)
        fn, user = C.cast(keep, C.c_void_p), None
    its = C.c_int(0)
    hcap = maxit + 64
    hist = np.zeros(hcap)
    hlen = C.c_int(0)
    fin = C.c_double(0)
    dg = np.zeros(3)
    if orth not in ("cgs2", "dcgs2"):
        raise ValueError(f"orth must be 'cgs2' or 'dcgs2', not {orth!r}")
    fg = lib().or_fgmres if orth == "cgs2" else lib().or_fgmres_dcgs2
    st = fg(cplx, n, _p(rp), _p(ci), _p(v), fn, user, _p(b), _p(x), float(rtol), int(restart),
                         int(maxit), C.byref(its), hist.ctypes.data_as(C.POINTER(C.c_double)), hcap,
                         C.byref(hlen), C.byref(fin), int(diag), dg.ctypes.data_as(C.POINTER(C.c_double)))
    del keep
    out = dict(x=x, its=its.value, hist=hist[:hlen.value].copy(), final_relres=fin.value, status=st)
    if diag:
        out.update(orth=dg[0], arnoldi=dg[1], est_gap=dg[2])
    return out
