"""Accuracy of the tcgen05 conv path vs SIMT fp32 and the oracle: python tools/convacc.py L n"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from oracle import oracle as O  # noqa: E402
from paper_2203_11025_b200 import helmgpu as hg  # noqa: E402


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


L, n = int(sys.argv[1]), int(sys.argv[2])
rng = np.random.default_rng(3)
ctx = hg.Context(0)
kap = 0.1 + 0.3 * rng.random((n, n))
ctx.set_problem(kap, np.zeros((n, n)), 1.0, 0.0, 1.0)
ctx.build_hierarchy(hg.VCycleConfig(levels=2))
ctx.set_net(0, "solver", L, 16, 3, 0)
ctx.init_net_he(0, 9)
x = rng.standard_normal((2, 3, n, n)).astype(np.float32)
y_tc = ctx.net_forward(x)
ctx.set_option("tc_conv", 0)
y_simt = ctx.net_forward(x)
y_o = O.UNet(0, L, 16, 3, 0, seed=9).forward(x)
print(f"L={L} n={n} HB_CONV_DEBUG={os.environ.get('HB_CONV_DEBUG', '0')}: tc-vs-simt {rel(y_tc, y_simt):.2e} "
      f"tc-vs-oracle {rel(y_tc, y_o):.2e} simt-vs-oracle {rel(y_simt, y_o):.2e}")
