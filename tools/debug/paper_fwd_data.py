"""Paper U-Net forward (UNetConfig() at 128^2, batch 16): whole-forward device
time for different input data (checks data-dependent kernel speed)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2203_11025_b200 import helmgpu as hg  # noqa: E402

B, n = 16, 128
c = hg.Context(0)
c.set_paper_net(hg.UNetConfig(), "standalone")
for name, dims in c.paper_params():
    if name.endswith(".count"):
        c.paper_param(name, np.ones(dims, np.float32))
rng = np.random.default_rng(0)
z0, n0 = np.zeros((B, 4, n, n)), rng.standard_normal((B, 4, n, n))
warm = int(os.environ.get("WARM", "0"))
for lab, x in [("zeros", z0), ("normal", n0), ("zeros", z0), ("normal", n0), ("normal", n0), ("zeros", z0)]:
    x = x.astype(np.float32)
    for _ in range(1 + warm):
        c.paper_forward(x)
    c.prof_enable(True)
    c.prof_detail(True)
    c.paper_forward(x)
    recs = c.prof_detail(False)
    c.prof_enable(False)
    par = [us for lab2, us, by, fl in recs if "par4" in lab2]
    print(f"{lab:12s} total {sum(r[1] for r in recs):8.1f} us   par4 layers {' '.join(f'{u:.1f}' for u in par)}")
# the same network inside M_JU (hb_precond_apply, kind "ju")
import bench  # noqa: E402
from paper_2203_11025_b200 import problems  # noqa: E402
cfg = bench.config_for("c0")
ctx, arr = problems.gpu_setup(cfg, device=0)
ctx.set_paper_net(hg.UNetConfig(), "standalone")
for name, dims in ctx.paper_params():
    if name.endswith(".count"):
        ctx.paper_param(name, np.ones(dims, np.float32))
r = rng.standard_normal((B, n, n)) + 1j * rng.standard_normal((B, n, n))
for lab, rr in [("ju normal", r), ("ju real", r.real + 0j), ("ju zeros", 0 * r)]:
    ctx.precond_apply("ju", rr)
    ctx.prof_enable(True)
    ctx.prof_detail(True)
    ctx.precond_apply("ju", rr)
    recs = ctx.prof_detail(False)
    ctx.prof_enable(False)
    par = [us for lab2, us, by, fl in recs if "par4" in lab2]
    print(f"{lab:12s} total {sum(r[1] for r in recs):8.1f} us   par4 layers {' '.join(f'{u:.1f}' for u in par)}")
