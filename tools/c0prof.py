"""Run a few c0 x R solves through the device-resident FGMRES, for ncu:
   python tools/c0prof.py [replicas] [solves]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2203_11025_b200 import helmgpu as hg  # noqa: E402
from paper_2203_11025_b200 import problems  # noqa: E402

R = int(sys.argv[1]) if len(sys.argv) > 1 else 148
S = int(sys.argv[2]) if len(sys.argv) > 2 else 2
opts = [a.split("=") for a in sys.argv[3:]]
cfg = bench.config_for("c0")
ctx, arr = problems.gpu_setup(cfg, device=0)
for k, v in opts:
    ctx.set_option(k, int(v))
Bh = np.ascontiguousarray(problems.rhs_block(arr)[bench.columns(cfg, 1, 0, R)])
dB = torch.from_numpy(Bh).cuda()
dX = torch.zeros_like(dB)
kc = hg.KrylovConfig(restart=cfg["restart"], max_iters=cfg["max_iters"], rel_tol=1e-6)
stream = torch.cuda.ExternalStream(ctx.stream)
ts = []
for _ in range(S):
    dX.zero_()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    ctx.fgmres_device(cfg["precond"], dB.data_ptr(), dX.data_ptr(), Bh.shape[0], kc, want_report=False)
    e1.record(stream)
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
print(f"c0 x{R} {' '.join(a for a in sys.argv[3:])}: " + " ".join(f"{t:.2f}" for t in ts) + " ms/solve-step, "
      f"{R / (min(ts) * 1e-3):.0f} solves/s")
