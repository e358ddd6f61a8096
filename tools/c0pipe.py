"""Experiment: G independent solver contexts (column groups) on their own streams,
driven from G host threads, so one group's latency-bound coarse solve overlaps
another group's bandwidth-bound legs / Krylov kernels.
   python tools/c0pipe.py [replicas] [groups] [solves] [opt=val ...]"""
import os
import sys
import threading

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2203_11025_b200 import helmgpu as hg  # noqa: E402
from paper_2203_11025_b200 import problems  # noqa: E402

R = int(sys.argv[1]) if len(sys.argv) > 1 else 148
G = int(sys.argv[2]) if len(sys.argv) > 2 else 2
S = int(sys.argv[3]) if len(sys.argv) > 3 else 3
opts = [a.split("=") for a in sys.argv[4:]]
cfg = bench.config_for("c0")
kc = hg.KrylovConfig(restart=cfg["restart"], max_iters=cfg["max_iters"], rel_tol=1e-6)
groups = []
for g in range(G):
    ctx, arr = problems.gpu_setup(cfg, device=0)
    for k, v in opts:
        ctx.set_option(k, int(v))
    n = R // G + (1 if g < R % G else 0)
    Bh = np.ascontiguousarray(problems.rhs_block(arr)[[0] * n])
    dB = torch.from_numpy(Bh).cuda()
    groups.append((ctx, dB, torch.zeros_like(dB), n, torch.cuda.ExternalStream(ctx.stream)))


def run(i):
    ctx, dB, dX, n, _ = groups[i]
    ctx.fgmres_device(cfg["precond"], dB.data_ptr(), dX.data_ptr(), n, kc, want_report=False)


for it in range(S):
    for ctx, dB, dX, n, st in groups:
        dX.zero_()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e0.record(groups[0][4])
    for _, _, _, _, st in groups[1:]:
        st.wait_event(e0)
    th = [threading.Thread(target=run, args=(i,)) for i in range(G)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    ends = []
    for _, _, _, _, st in groups:
        e = torch.cuda.Event(enable_timing=True)
        e.record(st)
        ends.append(e)
    torch.cuda.synchronize()
    ms = max(e0.elapsed_time(e) for e in ends)
    print(f"c0 x{R} groups={G} {' '.join(sys.argv[4:])}: {ms:.2f} ms, {R / (ms * 1e-3):.0f} solves/s", flush=True)
