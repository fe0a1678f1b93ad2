"""clock64 trace of block 0 of one down launch of k_tri_reg (debug): per-level timing."""
import sys, ctypes as C
import numpy as np, torch
sys.path.insert(0, '.')
from synth import problems as P
import paper_2205_03224_b200 as gm
name, ilu, level = sys.argv[1], sys.argv[2], int(sys.argv[3])
prob, b, xt, prm = P.make_config(name)
s = gm.Solver(prob.rowptr, prob.colidx, prob.values, prm['levels'], prm['subdomains'], 0, ilu=ilu, coords=prob.coords, device=0)
x = torch.rand(prob.n, dtype=s.torch_dtype, device='cuda')
s.apply_precond(x); torch.cuda.synchronize()
buf = torch.zeros(8 * 4096, dtype=torch.int64, device='cuda')
gm.lib().gemslr_debug_trace(C.c_void_p(buf.data_ptr()))
gm.lib().gemslr_debug_trace_level(level)
s.apply_precond(x); torch.cuda.synchronize()
gm.lib().gemslr_debug_trace(C.c_void_p(0))
a = buf.cpu().numpy().reshape(2, 2048, 8)
t0 = a[:, :, 0][a[:, :, 0] > 0].min()
for sw in range(2):
    r = a[sw]
    r = r[r[:, 0] > 0].astype(np.float64)
    if len(r) == 0:
        continue
    ent, acc, rel, end, rot, ldi = [r[:, i] - t0 for i in range(6)]
    lv, wp = r[:, 6], r[:, 7]
    nl = int(lv.max()) + 1
    print(f"sweep {'LU'[sw]}: slices {len(r)} levels {nl}; per level {(acc.max() - acc.min()) / nl:.0f} cyc")
    print(f"   rel->acc {np.median(acc - rel):.0f} (p90 {np.percentile(acc - rel, 90):.0f})  acc->end(stores) {np.median(end - acc):.0f}")
    print(f"   rel->data ready {np.median(rot - rel):.0f}  data->2 ring LDS done {np.median(ldi - rot):.0f}  -> acc {np.median(acc - ldi):.0f}")
    # critical chain per level: the slice whose acc is last in level v-1 -> release of v
    crit = []
    for v in range(1, nl):
        m0, m1 = lv == v - 1, lv == v
        if m0.any() and m1.any():
            crit.append((rel[m1].min() - acc[m0].max(), (acc - rel)[m1].max()))
    crit = np.array(crit)
    print(f"   per level: last acc(v-1) -> first release(v) median {np.median(crit[:, 0]):.0f}; slowest compute in level median {np.median(crit[:, 1]):.0f}")
    ns_per = np.bincount(lv.astype(int))
    print(f"   slices per level: mean {ns_per.mean():.1f} max {ns_per.max()}; frac of slices whose warp's next slice is next level: {np.mean([lv[i + 15] == lv[i] + 1 for i in range(len(lv) - 15)]):.2f}")
    gaps = []
    for v in range(1, nl):
        m0, m1 = lv == v - 1, lv == v
        if m0.any() and m1.any():
            gaps.append(rel[m1].min() - end[m0].max())
    print(f"   last end of level v-1 -> first release of v: median {np.median(gaps):.0f}")
    NW = 15
    g2, g3 = [], []
    for v in range(1, nl):
        m0 = np.where(lv == v - 1)[0]
        m1 = lv == v
        if len(m0) and m1.any() and m0.max() + NW < len(r):
            arr = np.array([ent[i + NW] for i in m0])
            g2.append(rel[m1].min() - arr.max())
            g3.append(arr.max() - end[m0].max())
    print(f"   last arrival (next enter) -> release: median {np.median(g2):.0f}; last end -> last arrival: median {np.median(g3):.0f}")
    nxt = np.array([ent[i + 1] - ldi[i] if i + 1 < len(r) else 0 for i in range(len(r))])
    print("   first 12 slices: level warp enter rel acc end")
    for i in range(12):
        print("     ", int(lv[i]), int(wp[i]), *[int(v) for v in (ent[i], rel[i], acc[i], end[i])])
