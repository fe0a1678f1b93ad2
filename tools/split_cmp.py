"""Per-level triangular-solve times of a config with the split form off / 2 / 4 CTAs per block
(tri_split 1, 2, 4), apply parity between them.  python tools/split_cmp.py [C5] [1,2,4]"""
import sys
import numpy as np
import torch
sys.path.insert(0, '.')
from synth import problems as P
import paper_2205_03224_b200 as gm

name = sys.argv[1] if len(sys.argv) > 1 else 'C5'
splits = [int(k) for k in (sys.argv[2].split(',') if len(sys.argv) > 2 else ['1', '2', '4'])]
prob, b, xt, prm = P.make_config(name)
ref = None
for sp in splits:
    s = gm.Solver(prob.rowptr, prob.colidx, prob.values, prm['levels'], prm['subdomains'], prm['rank'], ilu=prm['ilu'],
                  coords=prob.coords, device=0, tri_split=sp)
    torch.manual_seed(0)
    x = torch.rand(prob.n, dtype=s.torch_dtype, device='cuda')
    for _ in range(3):
        y = s.apply_precond(x)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        y = s.apply_precond(x)
    e1.record()
    torch.cuda.synchronize()
    t_apply = e0.elapsed_time(e1) / 10
    s.profile(True, reset=True)
    for _ in range(10):
        s.apply_precond(x)
    torch.cuda.synchronize()
    s.profile(False)
    st = s.stats()
    k = st['kernels']
    yc = y.cpu().numpy()
    if ref is None:
        ref = yc
    err = np.linalg.norm(yc - ref) / np.linalg.norm(ref)
    print(f"{name} tri_split={sp} split={[L['stage']['split'] for L in st['stages']]} nw={[L['stage']['reg_nw'] for L in st['stages']]} "
          f"apply {t_apply * 1e3:.1f} us (rel diff vs first {err:.1e})")
    print("   packs", [(p['Q'], p['max_levels'], p['imp_L'], p['exports']) for p in st['packs']])
    for c in ('trisolve_down', 'trisolve_up', 'trisolve_last'):
        print(f"   {c:14s} per apply {k[c]['ms'] * 100:8.1f} us  by level " + ' '.join(f"{v * 100:8.1f}" for v in k[c]['by_level']))
    s.close()
