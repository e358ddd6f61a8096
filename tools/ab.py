"""A/B timing of library options on one config (device-resident FGMRES, CUDA events).

  python tools/ab.py c0 "staged_legs=0" "staged_legs=1" ...
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2203_11025_b200 import helmgpu as hg, problems  # noqa: E402

name = sys.argv[1]
variants = sys.argv[2:] or [""]
cfg = problems.get(name)
if name != "c0":
    cfg["max_iters"] = 20
reps = int(os.environ.get("REPLICAS", "1"))
ctx, arr = problems.gpu_setup(cfg)
Bh = problems.rhs_block(arr)
import numpy as np  # noqa: E402
B = torch.from_numpy(np.concatenate([Bh] * reps)).cuda()
X = torch.zeros_like(B)
kc = hg.KrylovConfig(restart=cfg["restart"], max_iters=cfg["max_iters"])
stream = torch.cuda.ExternalStream(ctx.stream)
for v in variants:
    for kv in [x for x in v.split(",") if x]:
        k, val = kv.split("=")
        ctx.set_option(k, int(val))
    for _ in range(3):
        X.zero_()
        rep = ctx.fgmres_device(cfg["precond"], B.data_ptr(), X.data_ptr(), B.shape[0], kc)
    ts = []
    for _ in range(5):
        X.zero_()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        ctx.fgmres_device(cfg["precond"], B.data_ptr(), X.data_ptr(), B.shape[0], kc, want_report=False)
        e1.record(stream)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    it = max(rep.iterations)
    print(f"{name} x{B.shape[0]} [{v}] iters={it} ms/step={min(ts):.3f} us/iter={1e3 * min(ts) / it:.1f} "
          f"solves/s={B.shape[0] * 1e3 / min(ts):.1f}", flush=True)
