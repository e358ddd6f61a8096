"""Per-launch device time of the coarsest GMRES(10) at a 3-level hierarchy of
n^2 (coarse (n/4)^2) for B columns: cluster kernel vs multi-launch Krylov path.
   python tools/debug/coarse_bench.py [n] [B ...]"""
import math
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2203_11025_b200 import helmgpu as hg  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
Bs = [int(a) for a in sys.argv[2:]] or [8, 16]
om = 2 * math.pi * 1.5 * n / 10
ctx = hg.Context(0)
ctx.set_problem(hg.make_medium(n, n, 1234), hg.absorbing_layer(n, n, 16, 2 * om), om, 1 / 16, 1 / 2.25)
ctx.build_hierarchy(hg.VCycleConfig(levels=3))
nc = n // 4
for B in Bs:
    f = np.random.default_rng(0).standard_normal((B, nc, nc)) + 0j
    for opt in (1, 0):
        ctx.set_option("coarse_cluster", opt)
        ctx.coarse_solve(f)
        ctx.prof_reset()
        ctx.prof_enable(True)
        for _ in range(5):
            ctx.coarse_solve(f)
        ctx.prof_enable(False)
        p = ctx.prof()["coarse_solve"]
        print(f"n={n} coarse={nc}^2 B={B} cluster={opt}: {1e3 * p['ms'] / 5:.1f} us per coarse solve")
