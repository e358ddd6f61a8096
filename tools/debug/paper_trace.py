import os, sys
sys.path.insert(0, "/root/repo")
import numpy as np
import bench
from paper_2203_11025_b200 import helmgpu as hg, problems
cfg = bench.config_for("c0")
ctx, arr = problems.gpu_setup(cfg, device=0)
ctx.set_paper_net(hg.UNetConfig(), "standalone")
for name, dims in ctx.paper_params():
    if name.endswith(".count"):
        ctx.paper_param(name, np.ones(dims, np.float32))
n = cfg["n"]
r = (np.random.default_rng(0).standard_normal((16, n, n)) + 0j)
for k in range(2):
    print("=== apply", k, file=sys.stderr)
    ctx.precond_apply("ju", r)
x = np.random.default_rng(0).standard_normal((16, 4, n, n)).astype(np.float32)
c2 = hg.Context(0)
c2.set_paper_net(hg.UNetConfig(), "standalone")
for name, dims in c2.paper_params():
    if name.endswith(".count"):
        c2.paper_param(name, np.ones(dims, np.float32))
for k in range(2):
    print("=== forward", k, file=sys.stderr)
    c2.paper_forward(x)
