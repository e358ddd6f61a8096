"""Per-launch device times (library profiler, eager) of one preconditioner apply
of a BASELINE config's full RHS block, aggregated by label:
   python tools/debug/cfg_layers.py c3 [B] [opt=v,opt=v]"""
import collections
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2203_11025_b200 import problems  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c3"
cfg = bench.config_for(name)
B = int(sys.argv[2]) if len(sys.argv) > 2 and sys.argv[2] else cfg["B"]
ctx, arr = problems.gpu_setup(cfg, device=0)
for kv in (sys.argv[3].split(",") if len(sys.argv) > 3 else []):
    k, v = kv.split("=")
    ctx.set_option(k, int(v))
n = cfg["n"]
r = (np.random.default_rng(0).standard_normal((B, n, n)) + 0j).astype(np.complex64)
dr = torch.from_numpy(r).cuda()
dz = torch.zeros_like(dr)
kind = cfg["precond"]
ctx.precond_apply_device(kind, dr.data_ptr(), dz.data_ptr(), B)
torch.cuda.synchronize()
ctx.prof_enable(True)
ctx.prof_detail(True)
ctx.precond_apply_device(kind, dr.data_ptr(), dz.data_ptr(), B)
torch.cuda.synchronize()
recs = ctx.prof_detail(False)
ctx.prof_enable(False)
agg = collections.OrderedDict()
for lab, us, by, fl in recs:
    a = agg.setdefault(lab, [0, 0.0, 0.0])
    a[0] += 1
    a[1] += us
    a[2] += fl
tot = sum(v[1] for v in agg.values())
print(f"{name} B={B} {kind}: {tot / 1e3:.2f} ms over {len(recs)} launches")
for lab, (cnt, us, fl) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:30]:
    print(f"  {us / 1e3:8.3f} ms {100 * us / tot:5.1f}%  x{cnt:3d}  {fl / (us * 1e-6) / 1e12 if fl else 0:6.1f} TF/s  {lab}")
