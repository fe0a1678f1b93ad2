"""Several right-hand sides (NEXT-4): apply / SpMV time per right-hand side on a config."""
import sys
import torch
sys.path.insert(0, '.')
from synth import problems as P
import paper_2205_03224_b200 as gm
name = sys.argv[1] if len(sys.argv) > 1 else 'C5'
prob, b, xt, prm = P.make_config(name)
s = gm.Solver(prob.rowptr, prob.colidx, prob.values, prm['levels'], prm['subdomains'], prm['rank'], ilu=prm['ilu'],
              coords=prob.coords, device=0)
n = s.n_local
for nr in (1, 2, 4, 8):
    X = torch.rand((nr, n), dtype=s.torch_dtype, device='cuda')
    for _ in range(2):
        s.apply_precond_multi(X)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        s.apply_precond_multi(X)
    e1.record()
    torch.cuda.synchronize()
    ta = e0.elapsed_time(e1) / 5
    e0.record()
    for _ in range(5):
        s.spmv_multi(X)
    e1.record()
    torch.cuda.synchronize()
    tsp = e0.elapsed_time(e1) / 5
    print(f"{name} nrhs {nr}: apply {ta * 1e3:8.1f} us ({ta * 1e3 / nr:7.1f} per rhs)   spmv {tsp * 1e3:7.1f} us "
          f"({tsp * 1e3 / nr:6.1f} per rhs)", flush=True)
