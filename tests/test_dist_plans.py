"""Multi-rank host logic on the CPU: ownership, local layouts and
halo plans of the product's host-only planning contexts (device = -1), checked
(1) in process for 2-4 ranks and (2) with real message passing over a
world-size-2 gloo process group, by emulating the distributed SpMV / E / F
products with the exchanged values and comparing with the oracle's global
products.  No GPU is used."""
import os
import socket

import numpy as np
import pytest
import scipy.sparse as sp

import oracle
from oracle import dense as D
from synth import problems as P

gm = pytest.importorskip("paper_2205_03224_b200")


def plans(prob, G, levels=3, p=8):
    out = []
    for r in range(G):
        s = gm.Solver(prob.rowptr, prob.colidx, prob.values, levels, p, 0, coords=prob.coords, device=-1,
                      nranks=G, my_rank=r)
        out.append(s)
    return out


def structure_of(s, tmpdir):
    # the global structure is identical on every rank; read it from rank 0's host plan export
    # (export is single-rank only, so rebuild a 1-rank plan with the same inputs)
    s1 = gm.Solver(s.rowptr, s.colidx, s.values, s.params.levels, s.params.subdomains, 0,
                   coords=s.coords, device=-1)
    from tests.bundle_io import Bundle
    B = Bundle(s1.export(str(tmpdir)))
    return B.structure(), s1


@pytest.mark.parametrize("G", [2, 3, 4])
def test_ownership_and_halo_symmetry(tmp_path, G):
    prob = P.laplacian((14, 12, 10))
    p = 12 if G == 3 else 8
    ss = plans(prob, G, p=p)
    st, s1 = structure_of(ss[0], tmp_path)
    perm = st["perm"]
    n = prob.n
    # every natural row owned exactly once; local layouts are level-major
    allrows = np.concatenate([s.perm for s in ss])
    assert np.array_equal(np.sort(allrows), np.arange(n))
    iperm = np.empty(n, np.int64)
    iperm[perm] = np.arange(n)
    for s in ss:
        pos = iperm[s.perm]
        assert np.all(np.diff(pos) > 0)          # ascending global position = level-major
    # level-0 parts in contiguous rank ranges
    bl0 = st["blocks"][0]
    for r, s in enumerate(ss):
        pos = iperm[s.perm]
        lev0 = pos[pos < st["level_off"][1]]
        q = np.searchsorted(bl0, lev0, side="right") - 1
        assert np.all(q // (p // G) == r)
    Ah = D.permute_matrix(prob.scipy(), perm).tocsr()
    owner = np.empty(n, np.int64)
    for r, s in enumerate(ss):
        owner[iperm[s.perm]] = r
    o = st["level_off"]
    L = len(o) - 1
    cases = [("A", 0, 0, n, 0, n)] + [("E", l, o[l + 1], n, o[l], o[l + 1]) for l in range(L)] + \
            [("F", l, o[l], o[l + 1], o[l + 1], o[L]) for l in range(L)]
    for which, l, r0, r1, c0, c1 in cases:
        hp = [s.halo_plan(which, l) for s in ss]
        for g in range(G):
            for h in range(G):
                # what g sends to h is exactly what h receives from g, in the same order
                sg = np.split(hp[g]["sglob"], np.cumsum(hp[g]["send_counts"])[:-1])[h]
                rh = np.split(hp[h]["rglob"], np.cumsum(hp[h]["recv_counts"])[:-1])[g]
                assert np.array_equal(sg, rh), (which, l, g, h)
        # completeness: every exterior column of a rank's rows is received
        sub = Ah[r0:r1, :].tocoo()
        for g in range(G):
            rows = sub.row + r0
            m = (owner[rows] == g) & (sub.col >= c0) & (sub.col < c1) & (owner[sub.col] != g)
            need = np.unique(sub.col[m])
            assert np.array_equal(np.sort(hp[g]["rglob"]), need), (which, l, g)
            assert np.all(owner[hp[g]["rglob"]] != g)


def test_distributed_spmv_emulation(tmp_path):
    """y = A x assembled rank by rank from owned values + the halo of plan A."""
    prob = P.convdiff_upwind((12, 10, 9))
    G = 2
    ss = plans(prob, G, p=8)
    st, _ = structure_of(ss[0], tmp_path)
    perm = st["perm"]
    iperm = np.empty(prob.n, np.int64)
    iperm[perm] = np.arange(prob.n)
    Ah = D.permute_matrix(prob.scipy(), perm).tocsr()
    x = P.rhs_vector(prob.n, False, 4)           # natural order
    xh = x[perm]                                 # permuted order
    y_or = oracle.spmv(prob, x)[perm]
    for s in ss:
        hp = s.halo_plan("A")
        own = iperm[s.perm]
        avail = np.full(prob.n, np.nan)
        avail[own] = xh[own]
        avail[hp["rglob"]] = xh[hp["rglob"]]     # the received values
        y_loc = Ah[own] @ np.nan_to_num(avail, nan=np.inf)
        assert np.all(np.isfinite(y_loc))        # no row touched a value it does not have
        assert np.allclose(y_loc, y_or[own], rtol=0, atol=1e-13)


def _free_port():
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        return so.getsockname()[1]


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        prob = P.laplacian((12, 12, 8))
        s = gm.Solver(prob.rowptr, prob.colidx, prob.values, 3, 8, 0, coords=prob.coords, device=-1,
                      nranks=world, my_rank=rank)
        s1 = gm.Solver(prob.rowptr, prob.colidx, prob.values, 3, 8, 0, coords=prob.coords, device=-1)
        n = prob.n
        # global permuted position of every natural row (1-rank plan = global order)
        iperm = np.empty(n, np.int64)
        iperm[s1.perm] = np.arange(n)
        v = P.rhs_vector(n, False, 11)           # the same global vector on both ranks, permuted order below
        vp = np.empty(n)
        vp[iperm] = v
        ok = True
        for which, levels in (("A", [0]), ("E", [0, 1, 2]), ("F", [0, 1, 2])):
            for l in levels:
                try:
                    hp = s.halo_plan(which, l)
                except gm.GemslrError:
                    continue
                sends = np.split(hp["sglob"], np.cumsum(hp["send_counts"])[:-1])
                recvs = np.split(hp["rglob"], np.cumsum(hp["recv_counts"])[:-1])
                reqs, bufs = [], []
                for peer in range(world):
                    if peer == rank:
                        continue
                    if len(sends[peer]):
                        reqs.append(dist.isend(torch.from_numpy(vp[sends[peer]].copy()), peer))
                    if len(recvs[peer]):
                        b = torch.empty(len(recvs[peer]), dtype=torch.float64)
                        bufs.append((peer, b))
                        reqs.append(dist.irecv(b, peer))
                for r_ in reqs:
                    r_.wait()
                for peer, b in bufs:
                    ok &= bool(np.array_equal(b.numpy(), vp[recvs[peer]]))
        q.put((rank, ok, int(s.n_local)))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_halo_exchange():
    import multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p_ in ps:
        p_.start()
    res = [q.get(timeout=300) for _ in ps]
    for p_ in ps:
        p_.join(timeout=60)
    assert all(ok for _, ok, _ in res), res
    assert sum(nl for _, _, nl in res) == 12 * 12 * 8
