"""C4 (complex Helmholtz) with and without the complex ILU shift (NEXT-3): iterations and time."""
import sys, time
import torch
sys.path.insert(0, '.')
from synth import problems as P
import paper_2205_03224_b200 as gm
name = sys.argv[1] if len(sys.argv) > 1 else 'C4'
kw = {}
if len(sys.argv) > 2:
    kw['omega2h2'] = float(sys.argv[2])
if len(sys.argv) > 3:
    kw['damping'] = float(sys.argv[3])
for shift in (0.0, 0.05):
    prob, b, xt, prm = P.make_config(name, **kw)
    t0 = time.time()
    s = gm.Solver(prob.rowptr, prob.colidx, prob.values, prm['levels'], prm['subdomains'], prm['rank'], ilu=prm['ilu'],
                  coords=prob.coords, device=0, ilu_shift=shift)
    ts = time.time() - t0
    bd = s.to_local(torch.from_numpy(b).cuda().to(s.torch_dtype))
    torch.cuda.synchronize(); t = time.time()
    out = s.solve(bd, rtol=prm['rtol'], restart=prm['restart'], maxit=1000)
    torch.cuda.synchronize(); dt = time.time() - t
    print(name, kw, 'shift', shift, 'its', out['its'], 'status', out['status'], 'solve %.3fs' % dt, 'setup %.1fs' % ts,
          'final %.2e' % out['final_relres'], flush=True)
    s.close()
