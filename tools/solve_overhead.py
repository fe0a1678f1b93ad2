"""Time C5 solves of K = 1, 2, 3, 5, 10, 20 iterations (CUDA events, best of 5) to separate
the fixed per-solve cost (first residual, cycle end: closing pass, y solve, x update,
explicit residual, host round trips) from the per-iteration cost.

  python tools/solve_overhead.py [config] [cgs2|dcgs2]
"""
import sys
import torch
sys.path.insert(0, '.')
from synth import problems as P
import paper_2205_03224_b200 as gm

name = sys.argv[1] if len(sys.argv) > 1 else 'C5'
orth = sys.argv[2] if len(sys.argv) > 2 else 'dcgs2'
prob, b, xt, prm = P.make_config(name)
s = gm.Solver(prob.rowptr, prob.colidx, prob.values, prm['levels'], prm['subdomains'], prm['rank'], ilu=prm['ilu'],
              coords=prob.coords, device=0)
s.set_orthogonalization(orth)
bd = s.to_local(torch.from_numpy(b).cuda().to(s.torch_dtype))
s.solve(bd, rtol=1e-300, restart=prm['restart'], maxit=60)
st = torch.cuda.current_stream()
for K in (1, 2, 3, 5, 10, 20, 40):
    best = 1e30
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(st)
        s.solve(bd, rtol=1e-300, restart=prm['restart'], maxit=K)
        e1.record(st)
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    print(f"{name} [{orth}] K {K:3d}: {best:8.3f} ms  ({best / K:.4f} ms/iteration)", flush=True)
