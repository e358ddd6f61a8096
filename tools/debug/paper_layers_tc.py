"""Per-layer device time of the paper U-Net forward (UNetConfig() at 128^2,
batch 16): tensor-core vs SIMT."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2203_11025_b200 import helmgpu as hg  # noqa: E402

B, n = int(sys.argv[1]) if len(sys.argv) > 1 else 16, 128
opts = [kv.split("=") for kv in (sys.argv[2].split(",") if len(sys.argv) > 2 else [])]
x = np.random.default_rng(0).standard_normal((B, 4, n, n)).astype(np.float32)
for tc in (1, 0):
    c = hg.Context(0)
    c.set_paper_net(hg.UNetConfig(), "standalone")
    for name, dims in c.paper_params():
        if name.endswith(".count"):
            c.paper_param(name, np.ones(dims, np.float32))
    c.set_option("tc_conv", tc)
    for k, v in opts:
        c.set_option(k, int(v))
    c.paper_forward(x)
    c.prof_enable(True)
    c.prof_detail(True)
    c.paper_forward(x)
    recs = c.prof_detail(False)
    c.prof_enable(False)
    tot = sum(r[1] for r in recs)
    print(f"tc_conv={tc}: total {tot:.1f} us over {len(recs)} launches")
    for lab, us, by, fl in recs:
        if us > 5:
            print(f"   {us:8.1f} us {fl / (us * 1e-6) / 1e12 if fl else 0:6.1f} TF/s  {lab}")
    c.close()
