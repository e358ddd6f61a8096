import sys, os, math, numpy as np
sys.path.insert(0, "/root/repo")
from paper_2203_11025_b200 import helmgpu as hg
from paper_2203_11025_b200 import problems, configs
cfg = configs.CONFIGS["c0"]
ctx, arr = problems.gpu_setup(cfg)
r = np.random.default_rng(0).standard_normal((49, 128, 128)) + 0j
for _ in range(3):
    ctx.precond_apply("v", r)
