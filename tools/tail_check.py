"""Tail form (DESIGN 6b) vs the plain order: apply parity with the oracle and whole solves.

  GEMSLR_TAIL=0|1 python tools/tail_check.py C5 [C2 ...]
"""
import json
import os
import sys
import tempfile
import time

import numpy as np
import torch

sys.path.insert(0, '.')
from synth import problems as P
import paper_2205_03224_b200 as gm

for name in [a for a in sys.argv[1:] if not a.startswith('--')] or ['C5']:
    prob, b, xt, prm = P.make_config(name)
    t0 = time.time()
    s = gm.Solver(prob.rowptr, prob.colidx, prob.values, prm['levels'], prm['subdomains'], prm['rank'], ilu=prm['ilu'],
                  coords=prob.coords, device=0)
    st = s.stats()
    print(name, 'TAIL', os.environ.get('GEMSLR_TAIL', '1'), 'setup %.1fs' % (time.time() - t0), 'fill %.3f' % st['fill'])
    for l, L in enumerate(st['stages']):
        g = L['stage']
        print('  level', l, 'depth', g.get('depth_L'), g.get('depth_U'), 'split', g.get('split'), 'tail', json.dumps(g.get('tail')))
    x = torch.rand(s.n_local, dtype=s.torch_dtype, device='cuda')
    for _ in range(3):
        s.apply_precond(x)
    torch.cuda.synchronize()
    s.profile(True, reset=True)
    for _ in range(10):
        s.apply_precond(x)
    torch.cuda.synchronize()
    s.profile(False)
    k = s.stats()['kernels']
    print('  apply kernels (us per apply):', {kk: round(v['ms'] * 100, 1) for kk, v in k.items() if v['count']})
    if '--oracle' in sys.argv:
        import oracle
        from tests.bundle_io import Bundle
        with tempfile.TemporaryDirectory() as d:
            B = Bundle(s.export(d))
            stt = B.structure()
            Pc = oracle.Precond(prob, stt, ilu=(oracle.ILU0 if prm['ilu'] == 'ilu0' else oracle.ILUT, 1e-3, 10))
            for l in range(B.L):
                lr = B.lowrank(l)
                if lr is not None:
                    Pc.set_lowrank(l, lr[0], lr[2])
        r = P.rhs_vector(prob.n, prob.is_complex, 5)
        yg = s.apply_precond(torch.from_numpy(r).cuda()).cpu().numpy()     # both in the permuted order (as smoke())
        yo = Pc.apply(r)
        print('  apply parity rel err %.3e' % (np.linalg.norm(yg - yo) / np.linalg.norm(yo)))
    bd = s.to_local(torch.from_numpy(b).cuda().to(s.torch_dtype))
    s.solve(bd, rtol=prm['rtol'], restart=prm['restart'], maxit=3)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    out = s.solve(bd, rtol=prm['rtol'], restart=prm['restart'], maxit=1000)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    xg = s.to_natural(out['x']).cpu().numpy()
    true_rel = float(np.linalg.norm(b - prob.scipy() @ xg) / np.linalg.norm(b))
    print(f"  solve its {out['its']} status {out['status']} {ms:.1f} ms {ms / max(out['its'], 1):.3f} ms/it true rel {true_rel:.2e}")
    s.close()
