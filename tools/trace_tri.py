"""Clock64 trace of block 0 of the level-0 down trisolve (debug)."""
import sys, ctypes as C
import numpy as np, torch
sys.path.insert(0, '.')
from synth import problems as P
import paper_2205_03224_b200 as gm
name, ilu = sys.argv[1], sys.argv[2]
prob, b, xt, prm = P.make_config(name)
s = gm.Solver(prob.rowptr, prob.colidx, prob.values, prm['levels'], prm['subdomains'], 0, ilu=ilu, coords=prob.coords, device=0)
x = torch.rand(prob.n, dtype=s.torch_dtype, device='cuda')
s.apply_precond(x); torch.cuda.synchronize()
buf = torch.zeros(8 * 4096, dtype=torch.int64, device='cuda')
gm.lib().gemslr_debug_trace(C.c_void_p(buf.data_ptr()))
# only level 0 launch wanted: run apply; the last down launch overwrites -> use C_last? record all, keep first
s.apply_precond(x); torch.cuda.synchronize()
allb = buf.cpu().numpy()
t = allb[:4 * 4096].reshape(-1, 4)
fma = allb[4 * 4096:5 * 4096].astype(np.float64)
col0 = allb[5 * 4096:6 * 4096].astype(np.float64)
n = int((t[:, 0] > 0).sum())
t = t[:n].astype(np.float64)
t0 = t[0, 0]
t -= t0
wait = t[:, 1] - t[:, 0]
comp = t[:, 2] - t[:, 1]
per = np.diff(t[:, 0])
print('chunks', n, 'total cycles %.0f' % t[-1, 2])
print('per-chunk cycles: median %.0f mean %.0f' % (np.median(per), per.mean()))
print('wait(full) median %.0f mean %.0f; compute median %.0f mean %.0f' % (np.median(wait), wait.mean(), np.median(comp), comp.mean()))
lead = t[:, 1] - t[:, 3]   # consumer got data minus producer issue time
print('issue->consumed: median %.0f' % np.median(lead))
nn = n
fm = fma[:nn] - t0
c0 = col0[:nn] - t0
ok = (fma[:nn] > 0) & (col0[:nn] > 0)
print('full_ok->col0 median %.0f ; col0->fma_done median %.0f ; fma_done->computed median %.0f' % (
    np.median((c0 - t[:, 1])[ok]), np.median((fm - c0)[ok]), np.median((t[:, 2] - fm)[ok])))
print('first 12 rows (start, full_ok, computed, issued):')
print(t[:12].astype(int))
