"""Trace of the split triangular solve (build with GEMSLR_TRACE=1): CTAs of block 0 of one
DOWN launch of a level, per slice clock64 before the level wait / after the import wait /
after the solve.  python tools/trace_split.py C5 0 [tri_split]"""
import sys, ctypes as C
import numpy as np, torch
sys.path.insert(0, '.')
from synth import problems as P
import paper_2205_03224_b200 as gm
name, level = sys.argv[1], int(sys.argv[2])
sp = int(sys.argv[3]) if len(sys.argv) > 3 else 0
prob, b, xt, prm = P.make_config(name)
s = gm.Solver(prob.rowptr, prob.colidx, prob.values, prm['levels'], prm['subdomains'], 0, ilu=prm['ilu'],
              coords=prob.coords, device=0, tri_split=sp)
Q = s.stats()['stages'][level]['stage']['split']
x = torch.rand(prob.n, dtype=s.torch_dtype, device='cuda')
s.apply_precond(x); torch.cuda.synchronize()
buf = torch.zeros(16 + 4 * 2 * 2048 * 4, dtype=torch.int64, device='cuda')
gm.lib().gemslr_debug_trace(C.c_void_p(buf.data_ptr()))
gm.lib().gemslr_debug_trace_level(level)
s.apply_precond(x); torch.cuda.synchronize()
gm.lib().gemslr_debug_trace(C.c_void_p(0))
a = buf.cpu().numpy()
hdr = a[:16].reshape(8, 2)
tr = a[16:].reshape(4, 2, 2048, 4)
g0 = hdr[:Q, 1].min()
print(f"{name} level {level}: Q = {Q}; CTA start (globaltimer ns rel): {[int(v - g0) for v in hdr[:Q, 1]]}")
for q in range(Q):
    for sw in range(2):
        r = tr[q, sw]
        r = r[r[:, 2] > 0].astype(np.int64)
        if len(r) == 0:
            continue
        c0 = hdr[q, 0]
        t0, t1, t2 = r[:, 0] - c0, r[:, 1] - c0, r[:, 2] - c0
        lv = r[:, 3] & 0xffffffff
        nd = r[:, 3] >> 32
        nl = int(lv.max()) + 1
        span = t2.max() - t0.min()
        wait = t1 - t0
        comp = t2 - t1
        print(f"  cta {q} sweep {'LU'[sw]}: slices {len(r)} levels {nl} first {t0.min()} last {t2.max()} span {span} "
              f"({span / max(nl, 1):.0f}/level); wait med {np.median(wait):.0f} p90 {np.percentile(wait, 90):.0f}; "
              f"solve med {np.median(comp):.0f}; need max {nd.max()}")

# consumer vs producer timing (L sweep: producer q-1; U sweep: producer q+1)
def sweep_rows(q, sw):
    r = tr[q, sw]
    r = r[r[:, 2] > 0].astype(np.int64)
    c0 = hdr[q, 0]
    return r[:, 0] - c0, r[:, 1] - c0, r[:, 2] - c0, r[:, 3] & 0xffffffff, r[:, 3] >> 32
for sw in range(2):
    for q in range(Q):
        p = q - 1 if sw == 0 else q + 1
        if p < 0 or p >= Q:
            continue
        t0, t1, t2, lv, nd = sweep_rows(q, sw)
        pt0, pt1, pt2, plv, pnd = sweep_rows(p, sw)
        pdone = {}
        for u in np.unique(plv):
            pdone[int(u)] = pt2[plv == u].max()
        rows = []
        for j in np.unique(lv)[:: max(1, len(np.unique(lv)) // 12)]:
            m = lv == j
            need = int(nd[m].max()) - 1
            rows.append((int(j), need, int(pdone.get(need, -1)), int(t0[m].min()), int(t1[m].max()), int(t2[m].max())))
        print(f"  {'LU'[sw]} consumer {q} <- producer {p}: (level, needs producer level, its done, enter, passed wait, done)")
        for r_ in rows:
            print("     ", r_)
