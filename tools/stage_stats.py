"""Print per-stage statistics (depth, cps, nnz) and per-kernel apply timing for a config."""
import json, sys, time
import numpy as np, torch
sys.path.insert(0, '.')
from synth import problems as P
import paper_2205_03224_b200 as gm
name = sys.argv[1] if len(sys.argv) > 1 else 'C5'
for ilu in sys.argv[2:] or ['ilut', 'ilu0']:
    prob, b, xt, prm = P.make_config(name)
    t = time.time()
    s = gm.Solver(prob.rowptr, prob.colidx, prob.values, prm['levels'], prm['subdomains'], prm['rank'], ilu=ilu,
                  coords=prob.coords, device=0)
    st = s.stats()
    print(name, ilu, 'setup %.1fs' % (time.time() - t), 'host %.1f dev %.1f arnoldi %.1f' % (st['setup_host_s'], st['setup_device_s'], st['arnoldi_s']))
    for l, L in enumerate(st['stages']):
        print(' level', l, json.dumps(L))
    print(' last', json.dumps(st['last']))
    x = torch.rand(prob.n, dtype=torch.float64, device='cuda')
    for _ in range(3): s.apply_precond(x)
    torch.cuda.synchronize()
    s.profile(True, reset=True)
    for _ in range(10): s.apply_precond(x)
    torch.cuda.synchronize()
    s.profile(False)
    print(' kernels', json.dumps(s.stats()['kernels']))
    s.close()
