"""Per-layer conv timing of a classic U-Net forward (library profiler, eager launches).

  python tools/convbench.py L n B [option=value ...]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2203_11025_b200 import helmgpu as hg  # noqa: E402

L, n, B = (int(a) for a in (sys.argv[1:4] if len(sys.argv) > 3 else (4, 128, 8)))
opts = sys.argv[4:]
ctx = hg.Context(0)
rng = np.random.default_rng(0)
ctx.set_problem(0.1 + 0.3 * rng.random((n, n)), np.zeros((n, n)), 1.0, 0.0, 1.0)
ctx.build_hierarchy(hg.VCycleConfig(levels=2))
ctx.set_net(0, "solver", L, 16, 3, 0)
ctx.init_net_he(0, 7)
for o in opts:
    k, v = o.split("=")
    ctx.set_option(k, int(v))
x = rng.standard_normal((B, 3, n, n)).astype(np.float32)
for _ in range(3):
    ctx.net_forward(x)
ctx.prof_enable(True)
ctx.prof_detail(True)
for _ in range(5):
    ctx.net_forward(x)
recs = ctx.prof_detail(False)
ctx.prof_enable(False)
agg = {}
order = []
for lab, us, by, fl in recs:
    if lab not in agg:
        order.append(lab)
    a = agg.setdefault(lab, [0, 0.0, fl])
    a[0] += 1
    a[1] += us
tot = sum(v[1] for v in agg.values()) / 5
flops = sum(v[2] * v[0] for v in agg.values()) / 5
print(f"L={L} n={n} B={B}: forward {tot:.1f} us (kernels summed), {flops / 1e9:.2f} GFLOP, "
      f"{flops / (tot * 1e-6) / 1e12:.1f} TFLOP/s")
for lab in order:
    cnt, us, fl = agg[lab]
    t = us / cnt
    print(f"  {lab:40s} {t:8.1f} us  {fl / (t * 1e-6) / 1e12 if fl else 0:7.1f} TFLOP/s  x{cnt // 5}")
