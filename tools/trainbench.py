"""Training throughput of the paper U-Net: one run_batch + adam_step per step
(UNetConfig() defaults, 128^2, batch 20 -- the paper's retraining batch), on the
device through the C ABI and on the reference (oracle/_ref, one host thread).

   python tools/trainbench.py [n] [batch] [steps] [--no-ref]
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2203_11025_b200 import helmgpu as hg  # noqa: E402

args = [a for a in sys.argv[1:] if not a.startswith("--")]
n = int(args[0]) if args else 128
B = int(args[1]) if len(args) > 1 else 20
steps = int(args[2]) if len(args) > 2 else 10
rs = np.random.default_rng(0)
x = rs.standard_normal((B, 4, n, n)).astype(np.float32)
x[:, :2] *= 1e-3
t = rs.standard_normal((B, 2, n, n)).astype(np.float32)
ctx = hg.Context(0)
ctx.set_paper_net(hg.UNetConfig(), "standalone")
ctx.paper_init(3)
for _ in range(2):
    ctx.paper_train_batch(x, t, step=True, lr=1e-5)
t0 = time.perf_counter()
for _ in range(steps):
    loss, _ = ctx.paper_train_batch(x, t, step=True, lr=1e-5)
dt = (time.perf_counter() - t0) / steps
print(f"device: {dt * 1e3:.2f} ms per batch of {B} at {n}^2 ({B / dt:.1f} samples/s), loss {loss:.4g}")
if "--no-ref" not in sys.argv:
    from oracle import oracle as O
    if O.have_ref():
        net = O.RefPaperNet(levels=3, base=16, rpl=1, bot=3, kud=5, kres=3, variant=0, seed=3)
        t0 = time.perf_counter()
        net.train_batch(x, t, step=True, lr=1e-5)
        dr = time.perf_counter() - t0
        print(f"reference (1 thread): {dr * 1e3:.1f} ms per batch ({B / dr:.2f} samples/s); device speed-up {dr / dt:.1f}x")
