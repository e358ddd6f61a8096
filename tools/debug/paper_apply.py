"""Whole M_JU applies with the paper U-Net (UNetConfig() at 128^2) on device c64
fields, CUDA events around back-to-back applies, per library option variant:
   python tools/debug/paper_apply.py [B] [opt=v,opt=v ...] ..."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2203_11025_b200 import helmgpu as hg  # noqa: E402
from paper_2203_11025_b200 import problems  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 16
cfg = bench.config_for("c0")
ctx, arr = problems.gpu_setup(cfg, device=0)
ctx.set_paper_net(hg.UNetConfig(), "standalone")
for name, dims in ctx.paper_params():
    if name.endswith(".count"):
        ctx.paper_param(name, np.ones(dims, np.float32))
n = cfg["n"]
r = np.random.default_rng(0).standard_normal((B, n, n)) + 1j * np.random.default_rng(1).standard_normal((B, n, n))
dr = torch.from_numpy(r.astype(np.complex64)).cuda()
dz = torch.zeros_like(dr)
stream = torch.cuda.ExternalStream(ctx.stream)
ref = None
for var in sys.argv[2:] or [""]:
    for kv in filter(None, var.split(",")):
        k, v = kv.split("=")
        ctx.set_option(k, int(v))
    ctx.precond_apply_device("ju", dr.data_ptr(), dz.data_ptr(), B)
    torch.cuda.synchronize()
    z = dz.cpu().numpy()
    ref = z if ref is None else ref
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(20):
        ctx.precond_apply_device("ju", dr.data_ptr(), dz.data_ptr(), B)
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 20
    print(f"{var or 'default':30s} B={B}: {1e3 * ms:8.1f} us per apply, {B / ms * 1e3:9.0f} applies/s, "
          f"rel vs first {np.linalg.norm(z - ref) / np.linalg.norm(ref):.1e}", flush=True)
