"""Solve a config to convergence with ILUT and ILU(0): iterations, time, true residual."""
import sys, time
import numpy as np, torch
sys.path.insert(0, '.')
from synth import problems as P
import paper_2205_03224_b200 as gm
name = sys.argv[1]
for ilu in sys.argv[2:] or ['ilut', 'ilu0']:
    prob, b, xt, prm = P.make_config(name)
    s = gm.Solver(prob.rowptr, prob.colidx, prob.values, prm['levels'], prm['subdomains'], prm['rank'], ilu=ilu,
                  coords=prob.coords, device=0)
    bd = s.to_local(torch.from_numpy(b).cuda().to(s.torch_dtype))
    s.solve(bd, rtol=prm['rtol'], restart=prm['restart'], maxit=3)
    torch.cuda.synchronize(); t = time.time()
    out = s.solve(bd, rtol=prm['rtol'], restart=prm['restart'], maxit=1000)
    torch.cuda.synchronize(); dt = time.time() - t
    print(name, ilu, 'its', out['its'], 'status', out['status'], 'time %.3fs' % dt, 'ms/it %.3f' % (1e3 * dt / max(out['its'], 1)),
          'final %.2e' % out['final_relres'], 'fill %.2f' % s.stats()['fill'], flush=True)
    s.close()
