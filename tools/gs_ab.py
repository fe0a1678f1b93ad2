"""Time the Gram-Schmidt kernels over one restart cycle of a config (per-kernel CUDA events;
cheap preconditioner: ILU(0), rank 0).  python tools/gs_ab.py C4 100"""
import sys
import torch
sys.path.insert(0, '.')
from synth import problems as P
import paper_2205_03224_b200 as gm
name = sys.argv[1] if len(sys.argv) > 1 else 'C4'
its = int(sys.argv[2]) if len(sys.argv) > 2 else 100
prob, b, xt, prm = P.make_config(name)
s = gm.Solver(prob.rowptr, prob.colidx, prob.values, prm['levels'], prm['subdomains'], 0, ilu='ilu0',
              coords=prob.coords, device=0)
bd = s.to_local(torch.from_numpy(b).cuda().to(s.torch_dtype))
s.solve(bd, rtol=1e-300, restart=its, maxit=3)
s.profile(True, reset=True)
out = s.solve(bd, rtol=1e-300, restart=its, maxit=its)
torch.cuda.synchronize()
s.profile(False)
k = s.stats()['kernels']['gs']
print(name, 'its', out['its'], 'gs ms', round(k['ms'], 3), 'launches', k['count'], 'ms per iteration', round(k['ms'] / its, 4))
