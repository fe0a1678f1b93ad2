"""Run a few preconditioner applications of a config (for ncu captures)."""
import sys
import torch
sys.path.insert(0, '.')
from synth import problems as P
import paper_2205_03224_b200 as gm
name, ilu, rank, reps = sys.argv[1], sys.argv[2], int(sys.argv[3]), int(sys.argv[4])
prob, b, xt, prm = P.make_config(name)
s = gm.Solver(prob.rowptr, prob.colidx, prob.values, prm['levels'], prm['subdomains'], rank, ilu=ilu,
              coords=prob.coords, device=0)
x = torch.rand(prob.n, dtype=s.torch_dtype, device='cuda')
for _ in range(reps):
    y = s.apply_precond(x)
torch.cuda.synchronize()
print('ok', s.stats()['stages'][0]['stage'])
