"""B200-native GeMSLR solve path (arXiv 2205.03224) — Python binding.

Argument marshalling only: every step of setup's device stage and of the solve
path (SpMV, preconditioner apply, Gram-Schmidt, FGMRES) runs in libgemslr.so
(include/gemslr.h).  PyTorch supplies device memory and the stream.  There is
no CPU fallback: importing this package without the built library raises.
"""
from __future__ import annotations

import ctypes as C
import json
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libgemslr.so")

_lib = None

GEMSLR_OK, GEMSLR_NOT_CONVERGED = 0, 1
STATUS = {0: "OK", 1: "NOT_CONVERGED", -1: "INVALID_ARG", -2: "BAD_CSR", -3: "PARTITION", -4: "ZERO_PIVOT",
          -5: "LOWRANK", -6: "STATE", -7: "CUDA", -8: "NCCL", -9: "OOM"}
ABI_FUNCTIONS = ["gemslr_create", "gemslr_nccl_unique_id", "gemslr_create_dist", "gemslr_create_hostcomm", "gemslr_halo_plan", "gemslr_set_allocator", "gemslr_set_coordinates", "gemslr_setup", "gemslr_layout",
                 "gemslr_spmv", "gemslr_apply_precond", "gemslr_spmv_multi", "gemslr_apply_precond_multi",
                 "gemslr_solve", "gemslr_set_orthogonalization", "gemslr_solve_host", "gemslr_to_local",
                 "gemslr_to_natural", "gemslr_export_setup", "gemslr_stats", "gemslr_profile", "gemslr_last_error",
                 "gemslr_destroy"]


def torch_empty_like(X):
    """an output block with the same (row) stride as X: the C-ABI takes one leading dimension"""
    import torch
    return torch.empty_strided(X.shape, X.stride(), dtype=X.dtype, device=X.device)


class GemslrError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"{STATUS.get(code, code)}: {msg}")
        self.code = code


class Params(C.Structure):
    _fields_ = [("levels", C.c_int), ("subdomains", C.c_int), ("rank", C.c_int), ("ilu", C.c_int),
                ("ilut_drop", C.c_double), ("ilut_fill", C.c_int), ("last_blocks", C.c_int),
                ("arnoldi_tol", C.c_double), ("arnoldi_max_cycles", C.c_int), ("seed", C.c_ulonglong),
                ("cluster_ctas", C.c_int), ("tri_kernel", C.c_int), ("root_inner_its", C.c_int),
                ("ilu_shift", C.c_double), ("tri_split", C.c_int)]


def lib():
    """Load libgemslr.so; raise loudly when it has not been built."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'` "
                              "(there is no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        vp, i64 = C.c_void_p, C.c_int64
        L.gemslr_create.argtypes = [C.POINTER(vp), C.c_int, vp, vp]
        L.gemslr_nccl_unique_id.argtypes = [C.c_char_p, vp]
        L.gemslr_create_dist.argtypes = [C.POINTER(vp), C.c_int, vp, C.c_int, C.c_int, vp, C.c_char_p]
        L.gemslr_halo_plan.argtypes = [vp, C.c_int, C.c_int, vp, vp, vp]
        L.gemslr_create_hostcomm.argtypes = [C.POINTER(vp), C.c_int, vp, C.c_int, C.c_int, _ALLRED, _SENDRECV, vp]
        L.gemslr_set_coordinates.argtypes = [vp, C.c_int, vp]
        L.gemslr_setup.argtypes = [vp, C.c_int, i64, vp, vp, vp, C.POINTER(Params)]
        L.gemslr_layout.argtypes = [vp, C.POINTER(i64), vp]
        L.gemslr_spmv.argtypes = [vp, vp, vp]
        L.gemslr_apply_precond.argtypes = [vp, vp, vp]
        L.gemslr_spmv_multi.argtypes = [vp, vp, vp, C.c_int, i64]
        L.gemslr_apply_precond_multi.argtypes = [vp, vp, vp, C.c_int, i64]
        sargs = [vp, vp, vp, C.c_double, C.c_int, C.c_int, C.POINTER(C.c_int), vp, C.c_int, C.POINTER(C.c_int),
                 C.POINTER(C.c_double)]
        L.gemslr_solve.argtypes = sargs
        L.gemslr_solve_host.argtypes = sargs
        L.gemslr_to_local.argtypes = [vp, vp, vp]
        L.gemslr_to_natural.argtypes = [vp, vp, vp]
        L.gemslr_export_setup.argtypes = [vp, C.c_char_p]
        L.gemslr_stats.argtypes = [vp, C.c_char_p, C.c_size_t]
        L.gemslr_profile.argtypes = [vp, C.c_int, C.c_int]
        L.gemslr_set_orthogonalization.argtypes = [vp, C.c_int]
        L.gemslr_last_error.argtypes = [vp]
        L.gemslr_last_error.restype = C.c_char_p
        L.gemslr_destroy.argtypes = [vp]
        L.gemslr_destroy.restype = None
        for f in ABI_FUNCTIONS:
            if f not in ("gemslr_last_error", "gemslr_destroy"):
                getattr(L, f).restype = C.c_int
        _lib = L
    return _lib


_ALLRED = C.CFUNCTYPE(C.c_int, C.c_void_p, C.POINTER(C.c_double), C.c_size_t)
_SENDRECV = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_int, C.POINTER(C.c_int), C.POINTER(C.POINTER(C.c_double)),
                        C.POINTER(C.c_size_t), C.POINTER(C.POINTER(C.c_double)), C.POINTER(C.c_size_t))


def _torch_host_callbacks():
    """Host-staged collectives over the default torch.distributed group (gloo)."""
    import torch
    import torch.distributed as dist

    def allreduce(_user, buf, count):
        try:
            t = torch.from_numpy(np.ctypeslib.as_array(buf, shape=(count,)))
            dist.all_reduce(t)
            return 0
        except Exception:
            return 1

    def sendrecv(_user, npeers, peers, sbufs, scounts, rbufs, rcounts):
        try:
            reqs = []
            for i in range(npeers):
                if scounts[i]:
                    reqs.append(dist.isend(torch.from_numpy(np.ctypeslib.as_array(sbufs[i], shape=(scounts[i],))), peers[i]))
                if rcounts[i]:
                    reqs.append(dist.irecv(torch.from_numpy(np.ctypeslib.as_array(rbufs[i], shape=(rcounts[i],))), peers[i]))
            for r in reqs:
                r.wait()
            return 0
        except Exception:
            return 1

    return _ALLRED(allreduce), _SENDRECV(sendrecv)


def nccl_lib_path():
    """libnccl.so.2 of the torch wheel (the one torch itself loads)."""
    try:
        import nvidia.nccl
        p = os.path.join(list(nvidia.nccl.__path__)[0], "lib", "libnccl.so.2")
        return p if os.path.exists(p) else None
    except Exception:
        return None


def _ptr(a):
    if a is None:
        return None
    if hasattr(a, "data_ptr"):
        return C.c_void_p(a.data_ptr())
    return a.ctypes.data_as(C.c_void_p)


class Solver:
    """setup(A, levels, k, rank) of the north star on one GPU.

    A: host CSR (rowptr int64, colidx int32, values float64/complex128), natural order.
    device = -1 builds a host-only planning context (no GPU calls).
    """

    def __init__(self, rowptr, colidx, values, levels, subdomains, rank, ilu="ilut", ilut_drop=1e-3,
                 ilut_fill=10, last_blocks=0, coords=None, device=0, stream=None, seed=0, arnoldi_tol=1e-2,
                 arnoldi_max_cycles=10, cluster_ctas=0, tri_kernel=0, ilu_shift=0.0, root_inner_its=0, nranks=None, my_rank=None, comm="nccl",
                 tri_split=0):
        """nranks/my_rank: None = single GPU, or taken from an initialised
        torch.distributed world (one process per GPU; the NCCL id is broadcast
        with torch.distributed).  device = -1 with explicit nranks/my_rank builds
        the host-only plan of that rank (no GPU, no NCCL).  comm = "host" uses the
        host-staged backend over torch.distributed (gloo) instead of NCCL.
        comm = "nccl1" on one GPU runs the distributed code path over a one-rank NCCL
        communicator (every all-reduce is an NCCL call; tests and the bench's
        distributed-path line)."""
        L = lib()
        self.rowptr = np.ascontiguousarray(rowptr, dtype=np.int64)
        self.colidx = np.ascontiguousarray(colidx, dtype=np.int32)
        self.is_complex = np.iscomplexobj(values)
        self.values = np.ascontiguousarray(values, dtype=np.complex128 if self.is_complex else np.float64)
        self.n = len(self.rowptr) - 1
        self.device = device
        self.h = C.c_void_p()
        if stream is None and device >= 0:
            import torch
            stream = torch.cuda.current_stream(device).cuda_stream
        if nranks is None and device >= 0:
            import torch.distributed as dist
            if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
                nranks, my_rank = dist.get_world_size(), dist.get_rank()
        self.nranks = nranks or 1
        self.my_rank = my_rank or 0
        if self.nranks == 1 and comm == "nccl1" and device >= 0:
            libp = nccl_lib_path()
            idb = C.create_string_buffer(128)
            self._check(L.gemslr_nccl_unique_id(libp.encode() if libp else None, idb), "nccl_unique_id")
            self._check(L.gemslr_create_dist(C.byref(self.h), int(device), C.c_void_p(stream or 0), 1, 0, idb,
                                             libp.encode() if libp else None), "create_dist")
        elif self.nranks == 1:
            self._check(L.gemslr_create(C.byref(self.h), int(device), None, C.c_void_p(stream or 0)), "create")
        elif comm == "host" and device >= 0:
            self._cbs = _torch_host_callbacks()
            self._check(L.gemslr_create_hostcomm(C.byref(self.h), int(device), C.c_void_p(stream or 0), self.nranks,
                                                 self.my_rank, self._cbs[0], self._cbs[1], None), "create_hostcomm")
        else:
            libp = nccl_lib_path()
            idb = C.create_string_buffer(128)
            if device >= 0:
                import torch
                import torch.distributed as dist
                if self.my_rank == 0:
                    self._check(L.gemslr_nccl_unique_id(libp.encode() if libp else None, idb), "nccl_unique_id")
                obj = [bytes(idb.raw)]
                dist.broadcast_object_list(obj, src=0)
                C.memmove(idb, obj[0], 128)
            self._check(L.gemslr_create_dist(C.byref(self.h), int(device), C.c_void_p(stream or 0), self.nranks,
                                             self.my_rank, idb if device >= 0 else None,
                                             libp.encode() if libp else None), "create_dist")
        if coords is not None:
            self.coords = np.ascontiguousarray(coords, dtype=np.float64)
            self._check(L.gemslr_set_coordinates(self.h, self.coords.shape[1], _ptr(self.coords)), "coordinates")
        p = Params(levels, subdomains, rank, 0 if ilu == "ilu0" else 1, ilut_drop, ilut_fill, last_blocks,
                   arnoldi_tol, arnoldi_max_cycles, seed, cluster_ctas, tri_kernel, root_inner_its,
                   ilu_shift, tri_split)
        self.params = p
        self._check(L.gemslr_setup(self.h, 1 if self.is_complex else 0, self.n, _ptr(self.rowptr), _ptr(self.colidx),
                                   _ptr(self.values), C.byref(p)), "setup")
        nl = C.c_int64(0)
        self._check(L.gemslr_layout(self.h, C.byref(nl), None), "layout")
        self.n_local = nl.value
        self.perm = np.empty(self.n_local, dtype=np.int64)      # natural row of every local row
        self._check(L.gemslr_layout(self.h, C.byref(nl), _ptr(self.perm)), "layout")

    # ------------------------------------------------------------------ helpers
    def _check(self, rc, what):
        if rc < 0:
            msg = lib().gemslr_last_error(self.h).decode() if self.h else ""
            raise GemslrError(rc, f"{what}: {msg}")
        return rc

    @property
    def torch_dtype(self):
        import torch
        return torch.complex128 if self.is_complex else torch.float64

    def _vec(self, n=None):
        import torch
        return torch.empty(self.n_local if n is None else n, dtype=self.torch_dtype, device=f"cuda:{self.device}")

    def _dev(self, x, n=None):
        n = self.n_local if n is None else n
        assert x.is_cuda and x.dtype == self.torch_dtype and x.is_contiguous() and x.numel() == n, \
            "device vectors must be contiguous CUDA tensors of the solver dtype and length n_local"
        return x

    # ------------------------------------------------------------------ the path
    def spmv(self, x, y=None):
        x = self._dev(x)
        y = self._vec() if y is None else self._dev(y)
        self._check(lib().gemslr_spmv(self.h, _ptr(x), _ptr(y)), "spmv")
        return y

    def apply_precond(self, x, y=None):
        x = self._dev(x)
        y = self._vec() if y is None else self._dev(y)
        self._check(lib().gemslr_apply_precond(self.h, _ptr(x), _ptr(y)), "apply_precond")
        return y

    def _block(self, X):
        assert X.is_cuda and X.dtype == self.torch_dtype and X.dim() == 2 and X.shape[1] == self.n_local \
            and X.stride(1) == 1, "blocks are CUDA tensors of shape (nrhs, n_local), rows contiguous"
        return X

    def spmv_multi(self, X, Y=None):
        """Y[c] = A X[c] for every row c of the (nrhs, n_local) block X (A read once)."""
        X = self._block(X)
        Y = torch_empty_like(X) if Y is None else self._block(Y)
        assert Y.stride(0) == X.stride(0), "X and Y need the same leading dimension"
        self._check(lib().gemslr_spmv_multi(self.h, _ptr(X), _ptr(Y), X.shape[0], X.stride(0)), "spmv_multi")
        return Y

    def apply_precond_multi(self, X, Y=None):
        """Y[c] = M^{-1} X[c] for every row c of the (nrhs, n_local) block X (NEXT-4)."""
        X = self._block(X)
        Y = torch_empty_like(X) if Y is None else self._block(Y)
        assert Y.stride(0) == X.stride(0), "X and Y need the same leading dimension"
        self._check(lib().gemslr_apply_precond_multi(self.h, _ptr(X), _ptr(Y), X.shape[0], X.stride(0)),
                    "apply_precond_multi")
        return Y

    def set_orthogonalization(self, orth):
        """'cgs2' (c5, default) or 'dcgs2' (c5', reading Q38) for the solves that follow."""
        code = {"cgs2": 0, "dcgs2": 1}.get(orth)
        if code is None:
            raise ValueError(f"orth must be 'cgs2' or 'dcgs2', not {orth!r}")
        self._check(lib().gemslr_set_orthogonalization(self.h, code), "set_orthogonalization")
        self.orth = orth

    def solve(self, b, x0=None, rtol=1e-8, restart=50, maxit=1000, orth=None):
        if orth is not None:
            self.set_orthogonalization(orth)
        b = self._dev(b)
        x = self._vec().zero_() if x0 is None else self._dev(x0.clone())
        its, hl, fr = C.c_int(0), C.c_int(0), C.c_double(0)
        hist = np.zeros(maxit + 2)
        rc = self._check(lib().gemslr_solve(self.h, _ptr(b), _ptr(x), rtol, restart, maxit, C.byref(its), _ptr(hist),
                                            len(hist), C.byref(hl), C.byref(fr)), "solve")
        return dict(x=x, its=its.value, hist=hist[:hl.value].copy(), final_relres=fr.value, status=rc)

    def solve_host(self, b, x0=None, rtol=1e-8, restart=50, maxit=1000, out=None, orth=None):
        """End-to-end solve from host vectors in natural order (copies inside the call)."""
        if orth is not None:
            self.set_orthogonalization(orth)
        dt = np.complex128 if self.is_complex else np.float64
        b = np.ascontiguousarray(b, dtype=dt)
        x = out if out is not None else np.zeros(self.n, dtype=dt)
        if x0 is not None:
            x[:] = x0
        its, hl, fr = C.c_int(0), C.c_int(0), C.c_double(0)
        hist = np.zeros(maxit + 2)
        rc = self._check(lib().gemslr_solve_host(self.h, _ptr(b), _ptr(x), rtol, restart, maxit, C.byref(its),
                                                 _ptr(hist), len(hist), C.byref(hl), C.byref(fr)), "solve_host")
        return dict(x=x, its=its.value, hist=hist[:hl.value].copy(), final_relres=fr.value, status=rc)

    def to_local(self, x_nat, out=None):
        """natural-order global vector (length n) -> this rank's local vector"""
        out = self._vec() if out is None else out
        self._check(lib().gemslr_to_local(self.h, _ptr(self._dev(x_nat, self.n)), _ptr(out)), "to_local")
        return out

    def to_natural(self, x_loc, out=None):
        """local vector -> natural-order global vector (only owned entries written)"""
        out = self._vec(self.n).zero_() if out is None else out
        self._check(lib().gemslr_to_natural(self.h, _ptr(self._dev(x_loc)), _ptr(out)), "to_natural")
        return out

    def halo_plan(self, which, level=0):
        """which: 'A' (SpMV), 'E' or 'F' (level). Returns dict(send_counts, recv_counts, sglob, rglob)."""
        w = {"A": 0, "E": 1, "F": 2}[which]
        cnt = np.zeros(2 * self.nranks, dtype=np.int64)
        self._check(lib().gemslr_halo_plan(self.h, w, level, _ptr(cnt), None, None), "halo_plan")
        sg = np.zeros(max(int(cnt[:self.nranks].sum()), 1), dtype=np.int64)
        rg = np.zeros(max(int(cnt[self.nranks:].sum()), 1), dtype=np.int64)
        self._check(lib().gemslr_halo_plan(self.h, w, level, _ptr(cnt), _ptr(sg), _ptr(rg)), "halo_plan")
        return dict(send_counts=cnt[:self.nranks].copy(), recv_counts=cnt[self.nranks:].copy(),
                    sglob=sg[:int(cnt[:self.nranks].sum())], rglob=rg[:int(cnt[self.nranks:].sum())])

    def export(self, directory):
        self._check(lib().gemslr_export_setup(self.h, os.fsencode(directory)), "export")
        return directory

    def stats(self):
        buf = C.create_string_buffer(1 << 20)
        self._check(lib().gemslr_stats(self.h, buf, len(buf)), "stats")
        return json.loads(buf.value.decode())

    def profile(self, enable=True, reset=False):
        self._check(lib().gemslr_profile(self.h, int(enable), int(reset)), "profile")

    def close(self):
        if getattr(self, "h", None) and self.h.value:
            lib().gemslr_destroy(self.h)
            self.h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
