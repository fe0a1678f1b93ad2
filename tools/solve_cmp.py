"""Solve configs to convergence on the GPU and with the oracle on the same setup bundle:
iterations (GPU / oracle), GPU time to solution and ms per iteration, true residual.

  python tools/solve_cmp.py C2 C3 C4 C5 [--no-oracle] [--dcgs2]
"""
import os
import sys
import tempfile
import time

import numpy as np
import torch

sys.path.insert(0, '.')
from synth import problems as P
import paper_2205_03224_b200 as gm

names = [a for a in sys.argv[1:] if not a.startswith('--')] or ['C2', 'C3', 'C4', 'C5']
with_oracle = '--no-oracle' not in sys.argv
orth = 'dcgs2' if '--dcgs2' in sys.argv else 'cgs2'
for name in names:
    prob, b, xt, prm = P.make_config(name)
    t0 = time.time()
    s = gm.Solver(prob.rowptr, prob.colidx, prob.values, prm['levels'], prm['subdomains'], prm['rank'], ilu=prm['ilu'],
                  coords=prob.coords, device=0)
    setup = time.time() - t0
    bd = s.to_local(torch.from_numpy(b).cuda().to(s.torch_dtype))
    s.solve(bd, rtol=prm['rtol'], restart=prm['restart'], maxit=3, orth=orth)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    out = s.solve(bd, rtol=prm['rtol'], restart=prm['restart'], maxit=1000)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    xg = s.to_natural(out['x']).cpu().numpy()
    true_rel = float(np.linalg.norm(b - prob.scipy() @ xg) / np.linalg.norm(b))
    line = (f"{name} [{orth}] its {out['its']} status {out['status']} solve {ms:.1f} ms  {ms / max(out['its'], 1):.3f} ms/it  "
            f"true rel {true_rel:.2e} (rtol {prm['rtol']:g})  setup {setup:.1f}s  fill {s.stats()['fill']:.2f}  "
            f"split {[L['stage']['split'] for L in s.stats()['stages']]}")
    if with_oracle:
        import oracle
        from tests.bundle_io import Bundle
        with tempfile.TemporaryDirectory() as d:
            B = Bundle(s.export(d))
            st = B.structure()
            Pc = oracle.Precond(prob, st, ilu=(oracle.ILU0 if prm['ilu'] == 'ilu0' else oracle.ILUT, 1e-3, 10))
            for l in range(B.L):
                lr = B.lowrank(l)
                if lr is not None:
                    Pc.set_lowrank(l, lr[0], lr[2])
        t1 = time.time()
        ref = oracle.fgmres(prob, b, M=Pc, rtol=prm['rtol'], restart=prm['restart'], maxit=1000, orth=orth)
        line += f"  | oracle its {ref['its']} ({time.time() - t1:.0f}s, {oracle.get_threads()} threads)"
    print(line, flush=True)
    s.close()
