"""M_V FGMRES on a large grid for a fixed small budget (V-cycle leg profiling):
   python tools/legprof.py [n] [B] [iters] [opt=value ...]
   python tools/legprof.py c2|c3 [B] [iters] [opt=value ...]   (the config's own preconditioner, e.g. M_VU)"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2203_11025_b200 import helmgpu as hg  # noqa: E402
from paper_2203_11025_b200 import problems  # noqa: E402

B = int(sys.argv[2]) if len(sys.argv) > 2 else 16
its = int(sys.argv[3]) if len(sys.argv) > 3 else 4
if len(sys.argv) > 1 and sys.argv[1].startswith("c"):
    cfg = bench.config_for(sys.argv[1])
    cfg.update(B=B)
else:
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
    cfg = bench.config_for("c3")
    cfg.update(n=n, B=B, precond="v", net=None, enc=None)
pc = cfg["precond"]
arr = problems.problem_arrays(cfg)
ctx, arr = problems.gpu_setup(cfg, device=0, arr=arr)
for o in sys.argv[4:]:
    k, v = o.split("=")
    ctx.set_option(k, int(v))
Bh = np.ascontiguousarray(problems.rhs_block(arr)[:B])
dB = torch.from_numpy(Bh).cuda()
dX = torch.zeros_like(dB)
kc = hg.KrylovConfig(restart=its, max_iters=its, rel_tol=1e-6)
ctx.fgmres_device(pc, dB.data_ptr(), dX.data_ptr(), B, kc, want_report=False)
torch.cuda.synchronize()
ctx.prof_reset()
ctx.prof_enable(True)
ctx.fgmres_device(pc, dB.data_ptr(), dX.data_ptr(), B, kc, want_report=False)
ctx.prof_enable(False)
for k, v in ctx.prof().items():
    if v["launches"]:
        gbs = v["bytes"] / (v["ms"] / 1e3) / 1e9 if v["bytes"] else 0
        print(f"{k:16s} {v['ms']:8.3f} ms {v['launches']:4d} launches {gbs:8.0f} GB/s")
