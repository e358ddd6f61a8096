"""Per-class device time of one c0 M_V apply of B columns under library option
variants (eager, CUDA events per launch):
   python tools/debug/vc_classes.py [B] [opt=v,opt=v ...] ..."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np  # noqa: E402

import bench  # noqa: E402
from paper_2203_11025_b200 import problems  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 148
variants = sys.argv[2:] or [""]
cfg = bench.config_for("c0")
ctx, arr = problems.gpu_setup(cfg, device=0)
r = np.random.default_rng(0).standard_normal((B, 128, 128)) + 0j
ref = None
for var in variants:
    for kv in filter(None, var.split(",")):
        k, v = kv.split("=")
        ctx.set_option(k, int(v))
    z = ctx.precond_apply("v", r)
    if ref is None:
        ref = z
    ctx.prof_reset()
    ctx.prof_enable(True)
    for _ in range(10):
        ctx.precond_apply("v", r)
    ctx.prof_enable(False)
    p = ctx.prof()
    tot = sum(v["ms"] for v in p.values()) / 10
    print(f"{var or 'default':40s} total {1e3 * tot:7.1f} us  " + "  ".join(
        f"{k}:{1e3 * v['ms'] / max(1, v['launches']):.1f}us x{v['launches'] // 10}" for k, v in p.items() if v["launches"])
        + f"  rel vs first {np.linalg.norm(z - ref) / np.linalg.norm(ref):.1e}", flush=True)
