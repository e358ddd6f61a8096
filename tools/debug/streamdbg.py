"""Debug: row-streaming vs shared-memory V-cycle legs vs oracle on small grids."""
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np  # noqa: E402

from oracle import oracle as O  # noqa: E402
from paper_2203_11025_b200 import helmgpu as hg  # noqa: E402


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


for n, levels in [(32, 2), (32, 3), (64, 2), (64, 3), (128, 3), (96, 2), (48, 2), (16, 2)]:
    om = 2 * math.pi * 1.5 * n / 10
    k2 = hg.make_medium(n, n, 1234)
    g = hg.absorbing_layer(n, n, 4, 2 * om)
    ctx = hg.Context(0)
    ctx.set_problem(k2, g, om, 1 / 16, 1 / 2.25)
    ctx.build_hierarchy(hg.VCycleConfig(levels=levels))
    r = O.random_complex_normal(5, (2, n, n))
    z1 = ctx.precond_apply("v", r)
    ctx.set_option("stream_vcycle", 0)
    z2 = ctx.precond_apply("v", r)
    H = O.Hierarchy(k2, g, om, 1 / 16, 1 / 2.25, levels=levels)
    zo = O.Precond("v", H).apply(r)
    d = np.abs(z1 - z2)
    iy, ix = np.unravel_index(np.argmax(d[0]), d[0].shape)
    print(n, levels, "stream-vs-fused %.2e" % rel(z1, z2), "stream-vs-oracle %.2e" % rel(z1, zo),
          "fused-vs-oracle %.2e" % rel(z2, zo), "worst at", (iy, ix), flush=True)
