"""ncu-free per-layer device times of one U-Net forward via CUDA graphs is not
available here; this prints the kernel launch order of one forward for ncu runs:
   python tools/convlayers.py L n B [opt=val ...]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2203_11025_b200 import helmgpu as hg  # noqa: E402

L, n, B = (int(a) for a in sys.argv[1:4])
ctx = hg.Context(0)
rng = np.random.default_rng(0)
ctx.set_problem(0.1 + 0.3 * rng.random((n, n)), np.zeros((n, n)), 1.0, 0.0, 1.0)
ctx.build_hierarchy(hg.VCycleConfig(levels=2))
ctx.set_net(0, "solver", L, 16, 3, 0)
ctx.init_net_he(0, 7)
for o in sys.argv[4:]:
    k, v = o.split("=")
    ctx.set_option(k, int(v))
x = rng.standard_normal((B, 3, n, n)).astype(np.float32)
for _ in range(2):
    ctx.net_forward(x)
print("ok")
