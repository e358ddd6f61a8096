"""Debug: slab vs whole-grid FGMRES histories (c4-shaped, net coarse)."""
import sys, os, math
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
from test_slab import _problem, _ctx, _group, rel
from paper_2203_11025_b200 import helmgpu as hg
from oracle import oracle as O

n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
coarse = sys.argv[2] if len(sys.argv) > 2 else "net"
k2, g, om = _problem(n)
seed = 11 if coarse == "net" else None
whole = _ctx(hg, k2, g, om, 4, coarse, net_seed=seed)
whole2 = _ctx(hg, k2, g, om, 4, coarse, net_seed=seed)
cs = _group(hg, k2, g, om, 4, coarse, 2, net_seed=seed)
r = O.random_complex_normal(8, (1, n, n))
zw = whole.precond_apply("v", r)
zw2 = whole.precond_apply("v", r)
zs = cs[0].precond_apply_slab("v", r)
print("precond slab vs whole", rel(zs, zw), "whole rerun", rel(zw2, zw))
for restart in (20, 32):
    cfg = hg.KrylovConfig(restart=restart, max_iters=40)
    Xw, rw = whole.fgmres("v", r, cfg)
    Xw2, rw2 = whole2.fgmres("v", r, cfg)
    Xs, rs = cs[0].fgmres_slab("v", r, cfg)
    hw, hw2, hs = [np.asarray(x.residual_history[0]) for x in (rw, rw2, rs)]
    hw, hw2, hs = hw / hw[0], hw2 / hw2[0], hs / hs[0]
    print("restart", restart)
    for i in range(0, len(hw), 2):
        print(f"  {i:3d} whole {hw[i]:.6f} whole2 {hw2[i]:.6f} slab {hs[i]:.6f}")
