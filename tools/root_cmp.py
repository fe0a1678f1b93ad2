"""NEXT-1: FGMRES iterations and time with 0 / 3 / 5 root GMRES steps on a config."""
import sys, time
import torch
sys.path.insert(0, '.')
from synth import problems as P
import paper_2205_03224_b200 as gm
name = sys.argv[1] if len(sys.argv) > 1 else 'C5'
for its in (0, 3, 5):
    prob, b, xt, prm = P.make_config(name)
    s = gm.Solver(prob.rowptr, prob.colidx, prob.values, prm['levels'], prm['subdomains'], prm['rank'], ilu=prm['ilu'],
                  coords=prob.coords, device=0, root_inner_its=its)
    bd = s.to_local(torch.from_numpy(b).cuda().to(s.torch_dtype))
    s.solve(bd, rtol=prm['rtol'], restart=prm['restart'], maxit=3)
    torch.cuda.synchronize(); t = time.time()
    out = s.solve(bd, rtol=prm['rtol'], restart=prm['restart'], maxit=1000)
    torch.cuda.synchronize(); dt = time.time() - t
    print(name, 'root its', its, 'FGMRES its', out['its'], 'status', out['status'], 'solve %.3fs' % dt,
          'ms/it %.3f' % (1e3 * dt / max(out['its'], 1)), 'final %.2e' % out['final_relres'], flush=True)
    s.close()
