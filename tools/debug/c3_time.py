"""c3: FGMRES fixed budget vs bare preconditioner applies (device events)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2203_11025_b200 import helmgpu as hg  # noqa: E402
from paper_2203_11025_b200 import problems  # noqa: E402

cfg = bench.config_for("c3")
ctx, arr = problems.gpu_setup(cfg, device=0)
Bh = np.ascontiguousarray(problems.rhs_block(arr))
nb = Bh.shape[0]
dB = torch.from_numpy(Bh).cuda()
dX = torch.zeros_like(dB)
st = torch.cuda.ExternalStream(ctx.stream)


def timed(fn):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    fn()
    e1.record(st)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1)


for its in (1, 2, 4):
    kc = hg.KrylovConfig(restart=cfg["restart"], max_iters=its, rel_tol=1e-6)
    ctx.fgmres_device(cfg["precond"], dB.data_ptr(), dX.data_ptr(), nb, kc, want_report=False)
    dX.zero_()
    t = timed(lambda: ctx.fgmres_device(cfg["precond"], dB.data_ptr(), dX.data_ptr(), nb, kc, want_report=False))
    print(f"fgmres budget {its}: {t:.1f} ms", flush=True)
r = torch.zeros((nb, cfg["n"], cfg["n"]), dtype=torch.complex64, device="cuda").normal_()
z = torch.zeros_like(r)
ctx.precond_apply_device(cfg["precond"], r.data_ptr(), z.data_ptr(), nb)
t = timed(lambda: [ctx.precond_apply_device(cfg["precond"], r.data_ptr(), z.data_ptr(), nb) for _ in range(4)])
print(f"4 applies: {t:.1f} ms", flush=True)
