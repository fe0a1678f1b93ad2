"""Run one FGMRES cycle of `its` iterations of a config with a cheap preconditioner (ILU(0), rank 0)
(for ncu captures of the Gram-Schmidt kernels).  argv: its [config] [cgs2|dcgs2]"""
import sys
import torch
sys.path.insert(0, '.')
from synth import problems as P
import paper_2205_03224_b200 as gm
its = int(sys.argv[1]) if len(sys.argv) > 1 else 30
name = sys.argv[2] if len(sys.argv) > 2 else 'C5'
orth = sys.argv[3] if len(sys.argv) > 3 else 'cgs2'
prob, b, xt, prm = P.make_config(name)
s = gm.Solver(prob.rowptr, prob.colidx, prob.values, prm['levels'], prm['subdomains'], 0, ilu='ilu0',
              coords=prob.coords, device=0)
bd = s.to_local(torch.from_numpy(b).cuda().to(s.torch_dtype))
out = s.solve(bd, rtol=1e-300, restart=max(its, prm['restart']), maxit=its, orth=orth)
torch.cuda.synchronize()
print('its', out['its'])
