"""The distributed device path on ONE GPU: two ranks (two processes) share
cuda:0 and run the multi-GPU algorithm with the host-staged communication
backend (gloo).  Ranks only wait on each other on the host, never inside a
kernel.  Checks SpMV and k = 0 apply against the oracle element by element,
and a rank-k FGMRES solve (iterations, true residual)."""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        return so.getsockname()[1]


def _worker(rank, world, port, q, case):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2205_03224_b200 as gm
        import oracle
        from synth import problems as P
        from tests.bundle_io import Bundle
        import tempfile
        name, dims, p, k = case
        prob, b, xt, prm = P.make_config(name, dims=dims, subdomains=p, rank=k)
        kw = dict(ilu=prm["ilu"], coords=prob.coords)
        s = gm.Solver(prob.rowptr, prob.colidx, prob.values, prm["levels"], p, k, device=0, nranks=world,
                      my_rank=rank, comm="host", **kw)
        dt = s.torch_dtype
        res = {}
        x = P.rhs_vector(prob.n, prob.is_complex, 3)
        xl = torch.from_numpy(x[s.perm]).to("cuda:0", dtype=dt)          # this rank's rows, local layout
        y = s.spmv(xl).cpu().numpy()
        y_or = oracle.spmv(prob, x)
        res["spmv"] = float(np.abs(y - y_or[s.perm]).max() / np.abs(y_or).max())
        if k == 0:
            # oracle apply on the structure of a 1-rank plan (the global structure is rank-independent)
            s1 = gm.Solver(prob.rowptr, prob.colidx, prob.values, prm["levels"], p, 0, device=-1, **kw)
            with tempfile.TemporaryDirectory() as d:
                B = Bundle(s1.export(d))
                st = B.structure()
            Pc = oracle.Precond(prob, st, ilu=(oracle.ILU0 if prm["ilu"] == "ilu0" else oracle.ILUT, 1e-3, 10))
            r = P.rhs_vector(prob.n, prob.is_complex, 5)
            iperm = np.empty(prob.n, np.int64)
            iperm[st["perm"]] = np.arange(prob.n)
            yo = Pc.apply(r[st["perm"]])                                     # permuted order
            yg = s.apply_precond(torch.from_numpy(r[s.perm]).to("cuda:0", dtype=dt)).cpu().numpy()
            ref = yo[iperm[s.perm]]
            res["apply"] = float(np.linalg.norm(yg - ref))
            res["apply_ref"] = float(np.linalg.norm(ref))
        out = s.solve(torch.from_numpy(b[s.perm]).to("cuda:0", dtype=dt), rtol=prm["rtol"], restart=prm["restart"])
        xg = out["x"].cpu().numpy()
        full = torch.zeros(prob.n, dtype=torch.complex128 if prob.is_complex else torch.float64)
        full[torch.from_numpy(s.perm)] = torch.from_numpy(xg)
        dist.all_reduce(full)
        xs = full.numpy()
        res["its"] = out["its"]
        res["status"] = out["status"]
        res["true_rel"] = float(np.linalg.norm(b - oracle.spmv(prob, xs)) / np.linalg.norm(b))
        res["n_local"] = int(s.n_local)
        res["halo"] = s.stats()["halo_recv"]
        q.put((rank, res))
    except Exception as e:  # report, do not hang the parent
        import traceback
        q.put((rank, {"error": traceback.format_exc()}))
    finally:
        dist.destroy_process_group()


CASES = [("C5", (20, 20, 20), 8, 0), ("C3", (18, 16, 16), 8, 6), ("C4", (14, 14, 12), 8, 0)]


@pytest.mark.parametrize("case", CASES)
def test_two_ranks_on_one_gpu(case):
    import multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q, case)) for r in range(2)]
    for p_ in ps:
        p_.start()
    res = dict(q.get(timeout=600) for _ in ps)
    for p_ in ps:
        p_.join(timeout=60)
    for r in range(2):
        assert "error" not in res[r], res[r]["error"]
    name, dims, p, k = case
    n = int(np.prod(dims))
    assert res[0]["n_local"] + res[1]["n_local"] == n and res[0]["halo"] > 0
    for r in range(2):
        assert res[r]["spmv"] <= 1e-13
        if k == 0:
            tot = np.sqrt(res[0]["apply"] ** 2 + res[1]["apply"] ** 2)
            ref = np.sqrt(res[0]["apply_ref"] ** 2 + res[1]["apply_ref"] ** 2)
            assert tot <= 1e-10 * ref
        assert res[r]["status"] == 0
    from synth import problems as P
    rtol = P.CONFIGS[name]["rtol"]
    assert res[0]["its"] == res[1]["its"]
    assert res[0]["true_rel"] <= rtol
