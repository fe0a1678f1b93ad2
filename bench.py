#!/usr/bin/env python
"""Bench: FGMRES solve-phase ms/iteration of the GeMSLR path on B200 (BASELINE.json metric).

A "step" is one preconditioned FGMRES iteration (the whole hot path: SpMV,
one GeMSLR apply, CGS2 Gram-Schmidt, Givens update).  Workload: config C5 at
N=1 — 3D 7-point Laplacian 128^3, l_ev = 3, p = 32, ILUT(1e-3, 10), rank 20,
restart 50 — the per-GPU problem of the north star's weak-scaling target.
Timed region: exactly K iterations (solve with maxit = K and an unreachable
tolerance), inputs resident in HBM; the working set (matrix, factors,
Krylov basis ~2.4 GB) exceeds the 126 MB L2, so no flush is needed.

  python bench.py [--gpus N --steps K --warmup W] [--impl reference]

--gpus N > 1 without a torch.distributed environment re-launches itself under
torch.distributed.run with N ranks (one process per GPU, NCCL); under torchrun
WORLD_SIZE must equal N.  --impl reference times the plain CPU oracle (oracle/)
on bounded samples of the same workload on the host cores.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import tempfile
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from synth import problems as P  # noqa: E402

METRIC = "FGMRES solve-phase ms/iteration (HBM GB/s fraction in roofline)"
# the operator and right-hand side of each BASELINE config (synth/problems.py CONFIGS)
_OPER = {"C1": "2D 5-pt Poisson", "C2": "3D 7-pt Laplacian", "C3": "3D upwind convection-diffusion beta=(20,20,20)",
         "C4": "3D complex shifted Helmholtz omega^2 h^2=0.1", "C5": "3D 7-pt Laplacian"}
_DATA = {"C1": "seeded 5-pt Poisson, b uniform[-1,1]", "C2": "seeded 7-pt Laplacian, b = A x_true",
         "C3": "seeded upwind convection-diffusion, b uniform[-1,1]",
         "C4": "seeded complex shifted Helmholtz, b uniform[-1,1] + i uniform[-1,1]",
         "C5": "seeded 7-pt Laplacian, b = A x_true"}
UNIT = "ms/iteration"


def cpu_info():
    """CPU model, sockets, physical cores (the oracle's timing context)."""
    model, sockets = None, set()
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name") and model is None:
                model = line.split(":", 1)[1].strip()
            if line.startswith("physical id"):
                sockets.add(line.split(":", 1)[1].strip())
    except OSError:
        pass
    try:
        import psutil
        phys = psutil.cpu_count(logical=False) or os.cpu_count()
        mem = round(psutil.virtual_memory().total / 2**30, 1)
    except Exception:
        phys, mem = os.cpu_count(), None
    try:
        avail = len(os.sched_getaffinity(0))
    except Exception:
        avail = os.cpu_count()
    return {"model": model, "sockets": len(sockets) or 1, "physical_cores": phys, "logical_cpus_available": avail,
            "mem_gib": mem}


def oracle_threads():
    info = cpu_info()
    return max(1, min(info["physical_cores"] or 1, info["logical_cpus_available"] or 1)), info


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi sampling DURING the timed region (B200_PROFILING.md clocks line)."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu=0):
        self.gpu = gpu
        self.proc = None
        self.path = None

    def __enter__(self):
        try:
            fd, self.path = tempfile.mkstemp(suffix=".csv")
            os.close(fd)
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
            time.sleep(0.3)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.proc is not None:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        if self.proc is None or not self.path:
            return None
        rows = []
        for line in open(self.path):
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                rows.append(dict(sm=float(parts[1]), smax=float(parts[2]), hw=parts[5], hwt=parts[6],
                                 swt=parts[7], pcap=parts[8]))
            except ValueError:
                continue
        os.unlink(self.path)
        if not rows:
            return None
        load = [r for r in rows if r["sm"] > 500] or rows
        reasons = set()
        for r in load:
            for k, nm in (("hw", "hw_slowdown"), ("hwt", "hw_thermal_slowdown"), ("swt", "sw_thermal_slowdown"),
                          ("pcap", "sw_power_cap")):
                if r[k].lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": float(np.median([r["sm"] for r in load])), "sm_max_mhz": max(r["smax"] for r in rows),
                "reasons": sorted(reasons), "samples": len(rows)}


def algorithmic_bytes(stats, v, ld_iters, n, orth="cgs2", closing=()):
    """Algorithmic bytes per kernel class for the iterations executed.

    trisolve: every stored factor entry once (value v + int32 column 4), the U
    diagonal once, the right-hand side read and the solution written (2 v per row);
    the up sweep adds the F_l entries (v + 4) and the read-modify-write of y (2 v
    per row) plus the temporary (2 v per row).
    gs: CGS2 pass j reads (j+1) basis columns + w (v per element) and passes 2-3 write w;
    DCGS2 step j: the dot pass reads j columns + u_j + w, the update pass reads j columns
    + u_j + w and writes v_j and u_{j+1}; a cycle's closing dot pass reads j + 1 columns.
    """
    per = {}
    down = up = last = 0
    for st in stats["stages"]:
        S = st["stage"]
        t = S.get("tail")
        if t:
            # tail form (DESIGN 6b): DOWN reads L (L_hh + L_t|h) and U_tt with the tail's
            # diagonal, b1, writes t and z1 on the tail; UP reads L_tt, U (U_tt + U_h|t) with
            # every diagonal, F_l, t, writes and reads u on the tail, writes y1
            nz = t["nnz"]
            down += (nz[0] + nz[1] + nz[2]) * (v + 4) + t["rows"] * v + 2 * S["rows"] * v + t["rows"] * v
            up += (nz[4] + nz[2] + nz[3]) * (v + 4) + S["rows"] * v + st["nnzF"] * (v + 4) + 2 * S["rows"] * v \
                + 2 * t["rows"] * v
            continue
        fac = (S["nnz"] - S["rows"]) * (v + 4) + S["rows"] * v
        down += fac + 2 * S["rows"] * v
        up += fac + st["nnzF"] * (v + 4) + 5 * S["rows"] * v
    S = stats["last"]
    last = (S["nnz"] - S["rows"]) * (v + 4) + S["rows"] * v + 2 * S["rows"] * v
    per["trisolve_down"] = down
    per["trisolve_up"] = up
    per["trisolve_last"] = last
    nnz = stats.get("nnz_local", stats["nnz"])
    per["spmv"] = nnz * (v + 4) + 2 * n * v
    ew = 0
    wax = 0
    for st in stats["stages"]:
        k = st["k"]
        ew += st["nnzE"] * (v + 4) + 2 * st["s"] * v + k * st["s"] * v
        wax += k * st["s"] * v + 2 * st["s"] * v
    per["ew"] = ew
    per["waxpy"] = wax
    gs = 0
    for j in ld_iters:
        if orth == "dcgs2":
            gs += (2 * j + 6) * n * v
        else:
            gs += 3 * (j + 1) * n * v + 3 * n * v + 2 * n * v
    for j in closing:
        gs += (j + 1) * n * v
    per["gs_total"] = gs
    return per


def run_ours(args):
    import torch
    import paper_2205_03224_b200 as gm

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    name = args.config
    prob, b, xt, prm = P.make_config(name, gpus=world)  # C5: 128^3 per GPU, p = 32 per GPU (weak scaling)
    if args.ilu:
        prm["ilu"] = args.ilu
    t0 = time.time()
    s = gm.Solver(prob.rowptr, prob.colidx, prob.values, prm["levels"], prm["subdomains"], prm["rank"],
                  ilu=prm["ilu"], ilut_drop=prm["ilut_drop"], ilut_fill=prm["ilut_fill"], coords=prob.coords,
                  device=local, cluster_ctas=args.cluster_ctas)
    setup_s = time.time() - t0
    s.set_orthogonalization(args.orth)
    stream = torch.cuda.current_stream()
    bd = s.to_local(torch.from_numpy(b).to(f"cuda:{local}", dtype=s.torch_dtype))
    K, W = args.steps, args.warmup
    restart = prm["restart"]
    # warm-up: W iterations (untimed)
    s.solve(bd, rtol=1e-300, restart=restart, maxit=max(W, 1))
    torch.cuda.synchronize()

    def timed(profile, maxit=None):
        if profile:
            s.profile(True, reset=True)
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        out = s.solve(bd, rtol=1e-300, restart=restart, maxit=maxit or K)
        e1.record(stream)
        torch.cuda.synchronize()
        if profile:
            s.profile(False)
        ms = e0.elapsed_time(e1)
        if world > 1:
            t = torch.tensor([ms], device=f"cuda:{local}")
            torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
            ms = float(t.item())
        return ms, out

    with ClockSampler(local) as clk:
        ms, out = timed(False)
    clocks = clk.summary()
    its = out["its"]
    assert its == K, (its, K)
    ms_per = ms / its
    # the cost of an iteration grows with its column in the restart cycle (CGS2 reads
    # j + 1 basis vectors): one whole cycle of `restart` iterations, timed the same way
    cyc = [timed(False, maxit=restart)[0] for _ in range(3)]
    cycle = {"iterations": restart, "ms_per_iteration": round(min(cyc) / restart, 4),
             "ms_per_iteration_runs": [round(c / restart, 4) for c in cyc],
             "note": "whole restart cycles (columns 1..m), best of 3; value/ms_per_step cover the first K columns"}
    # per-kernel CUDA-event timing over a second identical timed region
    ms_prof, out2 = timed(True)
    stats = s.stats()
    kern = stats["kernels"]
    v = 16 if prob.is_complex else 8
    n = s.n_local
    iters_j = [j % restart for j in range(K)]
    ab = algorithmic_bytes(stats, v, iters_j, n, args.orth,
                           closing=[K % restart or restart] if args.orth == "dcgs2" else ())
    gb = {
        "trisolve_down": ab["trisolve_down"] * K, "trisolve_up": ab["trisolve_up"] * K,
        "trisolve_last": ab["trisolve_last"] * K, "spmv": ab["spmv"] * (K + 2),
        "ew": ab["ew"] * K, "waxpy": ab["waxpy"] * K, "gs": ab["gs_total"],
    }
    peak, peak_src = peaks()
    per_kernel = {}
    for kname, d in kern.items():
        if d["count"] == 0:
            continue
        rec = {"ms_total": round(d["ms"], 4), "launches": d["count"], "us_per_launch": round(1e3 * d["ms"] / d["count"], 2)}
        if kname in gb and d["ms"] > 0:
            gbs = gb[kname] / (d["ms"] * 1e-3) / 1e9
            rec.update(algorithmic_GB=round(gb[kname] / 1e9, 4), GBps=round(gbs, 1), frac=round(gbs / peak, 4))
        per_kernel[kname] = rec
    dom = max((k for k in per_kernel if k in gb), key=lambda k: per_kernel[k]["ms_total"])
    dd = per_kernel[dom]
    traffic, traffic_src = None, None                # DRAM bytes per launch, ncu capture of this bench command
    try:
        import glob
        caps = sorted(glob.glob(os.path.join(ROOT, "profiles", "r*_traffic.json")))
        if caps:
            with open(caps[-1]) as f:
                tj = json.load(f)
            traffic = tj.get(dom)
            traffic_src = f"profiles/{os.path.basename(caps[-1])} ({tj.get('_capture', 'ncu --set full of this command')})"
    except Exception:
        traffic = None
    roofline = {"bound": "hbm", "kernel": dom, "achieved": dd["GBps"], "peak": peak, "unit": "GB/s",
                "frac": dd["frac"], "traffic": round(traffic) if traffic else None, "traffic_source": traffic_src,
                "peak_source": peak_src,
                "bytes_per_launch": round(gb[dom] / dd["launches"]), "us_per_launch": dd["us_per_launch"]}
    # The triangular solves are bound by their level depth, not by HBM:
    # the latency account of the dominant class — level-barrier rounds per launch set
    # (the deepest block of every stage, L + U sweeps) and the SM cycles each took,
    # against the floor tools/ubench/levels.cu measures for one round (one dependent
    # gather + DFMA chain + barrier hand-off, ~250 cycles at 1-2 slices per level).
    if dom.startswith("trisolve") and dom != "trisolve_last":
        try:
            def _depth(g):
                t = g["stage"].get("tail")
                if t:
                    return sum(t["depth_up" if dom == "trisolve_up" else "depth_down"])
                return g["stage"]["depth_L"] + g["stage"]["depth_U"]
            depth = sum(_depth(st) for st in stats["stages"])
            per_set = dd["ms_total"] * 1e3 / (dd["launches"] / max(len(stats["stages"]), 1))   # us per apply
            mhz = (clocks or {}).get("sm_mhz") or 1965.0
            roofline["latency"] = {"levels_per_apply": depth, "us_per_apply": round(per_set, 1),
                                   "cycles_per_level": round(per_set * mhz / depth, 1),
                                   "floor_cycles_per_level": 250, "floor_source": "tools/ubench/levels.cu (K = 1-2)"}
        except Exception:
            pass
    launches = int(sum(d["count"] for d in kern.values()))
    # end-to-end: host vectors in natural order through gemslr_solve_host
    # inputs and outputs in pinned host memory (the copies run at link speed)
    bh_t = torch.from_numpy(np.ascontiguousarray(b)).pin_memory()
    xh_t = torch.zeros_like(bh_t).pin_memory()
    bh, xh = bh_t.numpy(), xh_t.numpy()
    s.solve_host(bh, rtol=1e-300, restart=restart, maxit=2, out=xh)      # first call allocates its staging
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    t1 = time.perf_counter()
    oute = s.solve_host(bh, rtol=1e-300, restart=restart, maxit=K, out=xh)
    e2e_ms = (time.perf_counter() - t1) * 1e3 / oute["its"]
    if world > 1:
        t = torch.tensor([e2e_ms], device=f"cuda:{local}")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        e2e_ms = float(t.item())
    e2e = {"value": round(e2e_ms, 4), "unit": UNIT, "h2d_bytes_per_step": round(bh.nbytes / K),
           "d2h_bytes_per_step": round(xh.nbytes / K), "h2d_bytes_total": bh.nbytes, "d2h_bytes_total": xh.nbytes}
    # the distributed code path at N = 1 (one-rank NCCL communicator: every all-reduce an
    # NCCL call, overlapped SpMV form, FGMRES graphs with their NCCL calls, no peers):
    # what the multi-GPU path costs per GPU before any communication volume
    dist_path = None
    if world == 1 and not args.no_dist_path:
        try:
            s2 = gm.Solver(prob.rowptr, prob.colidx, prob.values, prm["levels"], prm["subdomains"], prm["rank"],
                           ilu=prm["ilu"], ilut_drop=prm["ilut_drop"], ilut_fill=prm["ilut_fill"], coords=prob.coords,
                           device=local, comm="nccl1")
            s2.set_orthogonalization(args.orth)
            s2.solve(bd, rtol=1e-300, restart=restart, maxit=max(W, 1))
            torch.cuda.synchronize()
            a0 = s2.stats()["allreduces"]
            f0 = torch.cuda.Event(enable_timing=True)
            f1 = torch.cuda.Event(enable_timing=True)
            f0.record(stream)
            o2 = s2.solve(bd, rtol=1e-300, restart=restart, maxit=K)
            f1.record(stream)
            torch.cuda.synchronize()
            dist_path = {"ms_per_iteration": round(f0.elapsed_time(f1) / o2["its"], 4), "iterations": o2["its"],
                         "nccl_allreduces_per_iteration": round((s2.stats()["allreduces"] - a0) / o2["its"], 2),
                         "note": "distributed code path on this GPU over a one-rank NCCL communicator (no peers)"}
            s2.close()
        except Exception as e:                                     # report, keep the main line
            dist_path = {"error": str(e)[:200]}
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(prob, prm, s, b, args.cpu_iters, args.orth)
    line = {
        "metric": METRIC, "value": round(ms_per, 4), "unit": UNIT, "n_gpus": world, "steps": K, "warmup": W,
        "ms_per_step": round(ms_per, 4), "higher_is_better": False, "scaling": "weak", "vs_baseline": None,
        "dtype": "c128" if prob.is_complex else "f64", "data": f"synthetic ({_DATA[name]})",
        "config": {"workload": f"{name}: {_OPER[name]} {'x'.join(str(d) for d in prob.dims)} per GPU, "
                               f"l_ev={prm['levels']}, p={prm['subdomains']}, {prm['ilu'].upper()}(1e-3,10), "
                               f"rank={prm['rank']}, restart={restart}",
                   "n": n, "nnz": prob.nnz, "levels": stats["levels"], "fill": round(stats["fill"], 3),
                   "parallelism": "1 GPU" if world == 1 else f"subdomain row partition over {world} GPUs (NCCL send/recv halos, all-reduce)",
                   "l2": "working set (~2.4 GB) > 126 MB L2; no flush",
                   "setup_s": round(setup_s, 2), "timed_region": f"{K} FGMRES iterations (maxit=K, unreachable rtol)",
                   "orth": args.orth},
        "cycle": cycle, "roofline": roofline, "kernels": per_kernel,
        "ms_per_step_profiled": round(ms_prof / out2["its"], 4),
        "profiled_note": "per-kernel CUDA events around every launch of a second identical K-iteration solve "
                         "(no graphs, done flag read every iteration: no no-op launches)",
        "e2e": e2e, "gpu_launches": launches, "clocks": clocks,
    }
    if dist_path is not None:
        line["dist_path_n1"] = dist_path
    if cpu is not None:
        line["cpu_baseline"] = cpu
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


def cpu_baseline(prob, prm, s, b, iters, orth="cgs2"):
    """The oracle as it stands (C++ with OpenMP over independent work and fixed-order
    reductions), bounded sample: `iters` FGMRES iterations of the same workload on the
    same exported setup bundle, with all physical cores and with one thread."""
    import oracle
    from tests.bundle_io import Bundle
    nth, info = oracle_threads()
    with tempfile.TemporaryDirectory() as d:
        s.export(d)
        B = Bundle(d)
        st = B.structure()
        oracle.set_threads(nth)
        t0 = time.perf_counter()
        kind = oracle.ILU0 if prm["ilu"] == "ilu0" else oracle.ILUT
        Pc = oracle.Precond(prob, st, ilu=(kind, prm["ilut_drop"], prm["ilut_fill"]))
        for l in range(B.L):
            lr = B.lowrank(l)
            if lr is not None:
                Pc.set_lowrank(l, lr[0], lr[2])
        t_setup = time.perf_counter() - t0
        res = {}
        for nt, its in ((nth, iters), (1, max(iters // 2, 2))):
            oracle.set_threads(nt)
            t1 = time.perf_counter()
            out = oracle.fgmres(prob, b, M=Pc, rtol=1e-300, restart=prm["restart"], maxit=its, orth=orth)
            res[nt] = (1e3 * (time.perf_counter() - t1) / out["its"], out["its"])
    return {"value": round(res[nth][0], 2), "unit": UNIT, "cores": nth, "kind": "oracle",
            "sample": f"{res[nth][1]} FGMRES iterations of the same {prob.n}-row workload on the same setup bundle "
                      f"(oracle factor setup {t_setup:.1f}s excluded)",
            "threads": nth, "one_thread": {"value": round(res[1][0], 2), "iterations": res[1][1]},
            "cpu": info}


def run_reference(args):
    """--impl reference: the oracle timed on the host cores (rank 0 only)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import oracle
    from oracle import dense as D
    nth, info = oracle_threads()
    oracle.set_threads(nth)
    name = args.config
    prob, b, xt, prm = P.make_config(name, gpus=1)
    t0 = time.perf_counter()
    st = D.rcb_structure(prob.scipy(), prob.coords, prm["levels"], prm["subdomains"])
    kind = oracle.ILU0 if prm["ilu"] == "ilu0" else oracle.ILUT
    Pc = oracle.Precond(prob, st, ilu=(kind, prm["ilut_drop"], prm["ilut_fill"]))
    D.arnoldi_lowrank(Pc, prm["rank"], seed=0)
    setup = time.perf_counter() - t0
    K, W = args.steps, args.warmup
    oracle.fgmres(prob, b, M=Pc, rtol=1e-300, restart=prm["restart"], maxit=max(1, min(W, 1)), orth=args.orth)
    t1 = time.perf_counter()
    out = oracle.fgmres(prob, b, M=Pc, rtol=1e-300, restart=prm["restart"], maxit=K, orth=args.orth)
    dt = time.perf_counter() - t1
    val = 1e3 * dt / out["its"]
    line = {"impl": "reference", "metric": METRIC, "value": round(val, 2), "unit": UNIT, "n_gpus": args.gpus, "steps": out["its"],
            "warmup": W, "ms_per_step": round(val, 2), "higher_is_better": False, "scaling": "weak",
            "vs_baseline": None, "dtype": "c128" if prob.is_complex else "f64", "data": f"synthetic ({_DATA[name]})",
            "config": {"workload": f"{name} per-GPU problem {prob.dims}", "n": prob.n, "setup_s": round(setup, 1),
                       "orth": args.orth},
            "cpu_baseline": {"value": round(val, 2), "unit": UNIT, "cores": nth, "kind": "oracle", "cpu": info,
                             "sample": f"{out['its']} FGMRES iterations, oracle's own RCB structure, ILU and "
                                       f"one-cycle Arnoldi low rank (setup {setup:.0f}s excluded)"},
            "e2e": {"value": round(val, 2), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C5")
    ap.add_argument("--ilu", default=None)
    ap.add_argument("--cluster-ctas", type=int, default=0)
    ap.add_argument("--cpu-iters", type=int, default=10)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-dist-path", action="store_true")
    ap.add_argument("--orth", default="dcgs2", choices=["cgs2", "dcgs2"],
                    help="FGMRES orthogonalisation: CGS2 (c5) or DCGS2 (c5', reading Q38), both sides")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    world = os.environ.get("WORLD_SIZE")
    if world is None and args.gpus > 1:
        # one process per GPU: re-launch under torch.distributed.run (NCCL over NVLink)
        import socket
        with socket.socket() as so:
            so.bind(("127.0.0.1", 0))
            port = so.getsockname()[1]
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
        sys.exit(subprocess.call(cmd))
    if world is not None and int(world) != args.gpus:
        sys.exit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world} (one rank per GPU)")
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
