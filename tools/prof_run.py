"""Short, deterministic runs of one config for ncu (one process, one GPU).

  python tools/prof_run.py c0 [solves]      # full FGMRES solves
  python tools/prof_run.py c1 iters         # fixed iteration budget
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2203_11025_b200 import helmgpu as hg, problems  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c0"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
cfg = problems.get(name)
if name != "c0":
    cfg["max_iters"] = reps
    reps = 1
ctx, arr = problems.gpu_setup(cfg)
if os.environ.get("HB_NO_GRAPHS"):
    ctx.set_option("cuda_graphs", 0)
B = problems.rhs_block(arr)
R = int(os.environ.get("REPLICAS", "1"))
if R > 1:
    B = np.concatenate([B] * R)
kc = hg.KrylovConfig(restart=cfg["restart"], max_iters=cfg["max_iters"])
for r in range(reps):
    X, rep = ctx.fgmres(cfg["precond"], B, kc)
print(name, "iterations", rep.iterations, "converged", rep.converged)
