"""The distributed device path on ONE GPU: two ranks (two processes) share
cuda:0 and run the multi-GPU algorithm with the host-staged communication
backend (gloo).  Ranks only wait on each other on the host, never inside a
kernel.  Checks SpMV and the apply (k = 0 and rank k, with the distributed
low-rank bases gathered by the collective export) against the oracle element by
element, and an FGMRES solve (iterations, true residual)."""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        return so.getsockname()[1]


def _worker(rank, world, port, q, case, bdir):
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
        # the bundle of the distributed setup (collective; rank 0 writes, W_l gathered)
        s.export(bdir)
        dist.barrier()
        B = Bundle(bdir)
        st = B.structure()
        assert B.meta["nranks"] == world
        Pc = oracle.Precond(prob, st, ilu=(oracle.ILU0 if prm["ilu"] == "ilu0" else oracle.ILUT, 1e-3, 10))
        for l in range(B.L):
            lr = B.lowrank(l)
            if lr is not None:
                W, R, G = lr
                assert np.abs(W.conj().T @ W - np.eye(W.shape[1])).max() <= 1e-12     # c3.5 on the gathered W
                Pc.set_lowrank(l, W, G)
        res["k"] = [0 if B.lowrank(l) is None else B.lowrank(l)[0].shape[1] for l in range(B.L)]
        r = P.rhs_vector(prob.n, prob.is_complex, 5)
        iperm = np.empty(prob.n, np.int64)
        iperm[st["perm"]] = np.arange(prob.n)
        yo = Pc.apply(r[st["perm"]])                                         # permuted order
        yg = s.apply_precond(torch.from_numpy(r[s.perm]).to("cuda:0", dtype=dt)).cpu().numpy()
        ref = yo[iperm[s.perm]]
        res["apply"] = float(np.linalg.norm(yg - ref))
        res["apply_ref"] = float(np.linalg.norm(ref))
        # several right-hand sides on the distributed path (column by column, NEXT-4)
        r2 = P.rhs_vector(prob.n, prob.is_complex, 6)
        X = torch.stack([torch.from_numpy(r[s.perm]), torch.from_numpy(r2[s.perm])]).to("cuda:0", dtype=dt)
        Y = s.apply_precond_multi(X).cpu().numpy()
        ref2 = Pc.apply(r2[st["perm"]])[iperm[s.perm]]
        res["multi"] = float(max(np.linalg.norm(Y[0] - ref) / np.linalg.norm(ref),
                                 np.linalg.norm(Y[1] - ref2) / np.linalg.norm(ref2)))
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
        # DCGS2 across the two ranks (reading Q38): the dots / norm all-reduced between the
        # passes, the column and stopping steps as one-warp kernels; against the oracle's
        # fgmres_dcgs2 with the gathered bundle
        outd = s.solve(torch.from_numpy(b[s.perm]).to("cuda:0", dtype=dt), rtol=prm["rtol"], restart=prm["restart"],
                       orth="dcgs2")
        full.zero_()
        full[torch.from_numpy(s.perm)] = torch.from_numpy(outd["x"].cpu().numpy())
        dist.all_reduce(full)
        res["its_d"] = outd["its"]
        res["status_d"] = outd["status"]
        res["true_rel_d"] = float(np.linalg.norm(b - oracle.spmv(prob, full.numpy())) / np.linalg.norm(b))
        res["its_d_oracle"] = oracle.fgmres(prob, b, M=Pc, rtol=prm["rtol"], restart=prm["restart"], orth="dcgs2")["its"]
        q.put((rank, res))
    except Exception as e:  # report, do not hang the parent
        import traceback
        q.put((rank, {"error": traceback.format_exc()}))
    finally:
        dist.destroy_process_group()


CASES = [("C5", (20, 20, 20), 8, 0), ("C3", (18, 16, 16), 8, 6), ("C4", (14, 14, 12), 8, 5)]


@pytest.mark.parametrize("case", CASES)
def test_two_ranks_on_one_gpu(case, tmp_path):
    import multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q, case, str(tmp_path / "bundle"))) for r in range(2)]
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
        tot = np.sqrt(res[0]["apply"] ** 2 + res[1]["apply"] ** 2)
        ref = np.sqrt(res[0]["apply_ref"] ** 2 + res[1]["apply_ref"] ** 2)
        assert tot <= 1e-10 * ref, tot / ref
        assert res[r]["multi"] <= 1e-10
        if k > 0:
            assert min(res[r]["k"]) >= 1
        assert res[r]["status"] == 0
    from synth import problems as P
    rtol = P.CONFIGS[name]["rtol"]
    assert res[0]["its"] == res[1]["its"]
    assert res[0]["true_rel"] <= rtol
    assert res[0]["its_d"] == res[1]["its_d"] and res[0]["status_d"] == 0
    assert abs(res[0]["its_d"] - res[0]["its_d_oracle"]) <= 1, (res[0]["its_d"], res[0]["its_d_oracle"])
    assert res[0]["true_rel_d"] <= rtol


# ---------------------------------------------------------------- NCCL
def _pair(prob, prm, tmp_path, comm, tri_split=0):
    import paper_2205_03224_b200 as gm
    import oracle
    from tests.bundle_io import Bundle
    s = gm.Solver(prob.rowptr, prob.colidx, prob.values, prm["levels"], prm["subdomains"], prm["rank"],
                  ilu=prm["ilu"], coords=prob.coords, device=0, comm=comm, tri_split=tri_split)
    B = Bundle(s.export(str(tmp_path / f"bundle_{comm}")))
    st = B.structure()
    Pc = oracle.Precond(prob, st, ilu=(oracle.ILU0 if prm["ilu"] == "ilu0" else oracle.ILUT, 1e-3, 10))
    for l in range(B.L):
        lr = B.lowrank(l)
        if lr is not None:
            Pc.set_lowrank(l, lr[0], lr[2])
    return s, st, Pc


@pytest.mark.parametrize("name,dims,over,split", [("C3", (20, 18, 16), dict(subdomains=8, rank=6), 0),
                                                   ("C4", (16, 16, 14), dict(subdomains=8, rank=6), 0),
                                                   ("C5", (24, 24, 20), dict(subdomains=8, rank=4), 0),
                                                   ("C5", (28, 28, 24), dict(subdomains=4, rank=4), 4)])
def test_nccl_one_rank_distributed_path(tmp_path, name, dims, over, split):
    """The distributed code path (k_ew + NCCL all-reduce of W^H r + k_waxpy, the last
    separator gathered by an NCCL all-reduce and solved replicated, Gram-Schmidt dots
    all-reduced, FGMRES iterations captured as CUDA graphs WITH their NCCL calls) on
    one GPU over a one-rank NCCL communicator: apply parity with the oracle, FGMRES
    iterations within ±1 and the true residual, and NCCL calls actually made."""
    import torch
    import oracle
    from synth import problems as P
    prob, b, xt, prm = P.make_config(name, dims=dims, **over)
    s, st, Pc = _pair(prob, prm, tmp_path, "nccl1", tri_split=split)
    if split:
        assert s.stats()["stages"][0]["stage"]["split"] > 1
    dt = s.torch_dtype
    for seed in (2, 3):
        r = P.rhs_vector(prob.n, prob.is_complex, seed)
        yg = s.apply_precond(torch.from_numpy(r).to("cuda:0", dtype=dt)).cpu().numpy()
        yo = Pc.apply(r)
        assert np.linalg.norm(yg - yo) <= 1e-10 * np.linalg.norm(yo)
    a0 = s.stats()["allreduces"]
    out = s.solve(torch.from_numpy(b[st["perm"]]).to("cuda:0", dtype=dt), rtol=prm["rtol"], restart=prm["restart"])
    ref = oracle.fgmres(prob, b, M=Pc, rtol=prm["rtol"], restart=prm["restart"])
    assert out["status"] == 0 and abs(out["its"] - ref["its"]) <= 1, (out["its"], ref["its"])
    xg = np.empty(prob.n, dtype=b.dtype)
    xg[st["perm"]] = out["x"].cpu().numpy()
    assert np.linalg.norm(b - oracle.spmv(prob, xg)) <= prm["rtol"] * np.linalg.norm(b)
    st2 = s.stats()
    assert st2["nranks"] == 1 and st2["allreduces"] > a0          # the all-reduces went through NCCL
    # DCGS2 on the distributed path: dots and norm all-reduced between the passes, the
    # column / stopping steps as one-warp kernels (captured with the NCCL calls)
    a1 = st2["allreduces"]
    out = s.solve(torch.from_numpy(b[st["perm"]]).to("cuda:0", dtype=dt), rtol=prm["rtol"], restart=prm["restart"],
                  orth="dcgs2")
    ref = oracle.fgmres(prob, b, M=Pc, rtol=prm["rtol"], restart=prm["restart"], orth="dcgs2")
    assert out["status"] == 0 and abs(out["its"] - ref["its"]) <= 1, (out["its"], ref["its"])
    h = min(len(out["hist"]), len(ref["hist"]))
    assert np.allclose(out["hist"][:h], ref["hist"][:h], rtol=1e-6, atol=1e2 * prm["rtol"])
    xg[st["perm"]] = out["x"].cpu().numpy()
    assert np.linalg.norm(b - oracle.spmv(prob, xg)) <= prm["rtol"] * np.linalg.norm(b)
    assert s.stats()["allreduces"] > a1


def _nccl_worker(rank, world, port, q, case):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(rank)
    dist.init_process_group("gloo", rank=rank, world_size=world)     # only for the NCCL id broadcast
    try:
        import paper_2205_03224_b200 as gm
        import oracle
        from synth import problems as P
        name, dims, p, k = case
        prob, b, xt, prm = P.make_config(name, dims=dims, subdomains=p, rank=k)
        s = gm.Solver(prob.rowptr, prob.colidx, prob.values, prm["levels"], p, k, ilu=prm["ilu"], coords=prob.coords,
                      device=rank, nranks=world, my_rank=rank, comm="nccl")
        dt = s.torch_dtype
        x = P.rhs_vector(prob.n, prob.is_complex, 3)
        y = s.spmv(torch.from_numpy(x[s.perm]).to(f"cuda:{rank}", dtype=dt)).cpu().numpy()
        y_or = oracle.spmv(prob, x)
        res = {"spmv": float(np.abs(y - y_or[s.perm]).max() / np.abs(y_or).max())}
        out = s.solve(torch.from_numpy(b[s.perm]).to(f"cuda:{rank}", dtype=dt), rtol=prm["rtol"], restart=prm["restart"])
        full = torch.zeros(prob.n, dtype=torch.complex128 if prob.is_complex else torch.float64)
        full[torch.from_numpy(s.perm)] = torch.from_numpy(out["x"].cpu().numpy())
        dist.all_reduce(full)
        res.update(its=out["its"], status=out["status"],
                   true_rel=float(np.linalg.norm(b - oracle.spmv(prob, full.numpy())) / np.linalg.norm(b)))
        outd = s.solve(torch.from_numpy(b[s.perm]).to(f"cuda:{rank}", dtype=dt), rtol=prm["rtol"],
                       restart=prm["restart"], orth="dcgs2")                     # DCGS2 over NCCL (Q38)
        full.zero_()
        full[torch.from_numpy(s.perm)] = torch.from_numpy(outd["x"].cpu().numpy())
        dist.all_reduce(full)
        res.update(its_d=outd["its"], status_d=outd["status"],
                   true_rel_d=float(np.linalg.norm(b - oracle.spmv(prob, full.numpy())) / np.linalg.norm(b)))
        q.put((rank, res))
    except Exception:
        import traceback
        q.put((rank, {"error": traceback.format_exc()}))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("case", [("C3", (18, 16, 16), 8, 6), ("C4", (14, 14, 12), 8, 5)])
def test_two_ranks_nccl_two_gpus(case):
    """Two ranks on two GPUs over NCCL (send/recv halos, all-reduces); skipped with one GPU
    (two NCCL ranks must not share a GPU: kernels that wait on each other)."""
    import torch
    if torch.cuda.device_count() < 2:
        pytest.skip("needs two GPUs")
    import multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_nccl_worker, args=(r, 2, port, q, case)) for r in range(2)]
    for p_ in ps:
        p_.start()
    res = dict(q.get(timeout=600) for _ in ps)
    for p_ in ps:
        p_.join(timeout=60)
    for r in range(2):
        assert "error" not in res[r], res[r]["error"]
        assert res[r]["spmv"] <= 1e-13 and res[r]["status"] == 0
    from synth import problems as P
    assert res[0]["its"] == res[1]["its"]
    assert res[0]["true_rel"] <= P.CONFIGS[case[0]]["rtol"]
    assert res[0]["its_d"] == res[1]["its_d"] and res[0]["status_d"] == 0
    assert res[0]["true_rel_d"] <= P.CONFIGS[case[0]]["rtol"]
