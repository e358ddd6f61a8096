"""Per-layer device times of the paper U-Net inside M_JU (c0 grid, batch 16)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2203_11025_b200 import helmgpu as hg, problems
import bench
cfg = bench.config_for("c0")
ctx, arr = problems.gpu_setup(cfg)
ctx.set_paper_net(hg.UNetConfig(), "standalone")
for name, dims in ctx.paper_params():
    if name.endswith(".count"):
        ctx.paper_param(name, np.ones(dims, np.float32))
B = int(sys.argv[1]) if len(sys.argv) > 1 else 16
r = np.random.default_rng(0).standard_normal((B, 128, 128)) + 0j
ctx.precond_apply("ju", r)
ctx.prof_enable(True)
ctx.prof_detail(True)
ctx.precond_apply("ju", r)
ctx.prof_enable(False)
tot = 0
for lab, us, by, fl in ctx.prof_detail(False):
    tot += us
    print(f"{lab:28s} {us:8.1f} us  {fl / 1e9:7.3f} GFLOP  {fl / (us * 1e-6) / 1e12 if us > 0 else 0:6.2f} TF/s")
print("total", tot)
