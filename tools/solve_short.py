"""A short FGMRES solve of a config (for ncu launch lists): maxit iterations, unreachable rtol.  argv: config its [cgs2|dcgs2]"""
import sys
import torch
sys.path.insert(0, '.')
from synth import problems as P
import paper_2205_03224_b200 as gm
name, its = sys.argv[1], int(sys.argv[2])
ortho = sys.argv[3] if len(sys.argv) > 3 else 'cgs2'
prob, b, xt, prm = P.make_config(name)
s = gm.Solver(prob.rowptr, prob.colidx, prob.values, prm['levels'], prm['subdomains'], prm['rank'], ilu=prm['ilu'],
              coords=prob.coords, device=0)
bd = s.to_local(torch.from_numpy(b).cuda().to(s.torch_dtype))
out = s.solve(bd, rtol=1e-300, restart=prm['restart'], maxit=its, orth=ortho)
torch.cuda.synchronize()
print(name, 'its', out['its'])
