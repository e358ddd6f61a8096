"""Marginal cost of each kernel class in the c0 x 444 step (3 column groups,
as bench.py): every column runs exactly 105 FGMRES iterations (rel_tol 1e-12,
max_iters 105) and the option debug_skip drops kernel classes (results are
invalid; timing only).  bits: 1 level-0 legs, 2 level>=1 legs, 4 coarsest solve,
8 Krylov dots, 16 finalize.
   python tools/debug/c0_marginal.py [skip masks ...] [--opt k=v ...]"""
import os
import sys
import threading

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2203_11025_b200 import helmgpu as hg  # noqa: E402
from paper_2203_11025_b200 import problems  # noqa: E402

args = sys.argv[1:]
opts = [a.split("=") for a in args if "=" in a]
masks = [int(a) for a in args if "=" not in a] or [0, 1, 2, 4, 6, 8, 16, 7]
cfg = bench.config_for("c0")
G, R = 3, 444
bounds = [R * g // G for g in range(G + 1)]
groups = []
for g in range(G):
    cg, arr = problems.gpu_setup(cfg, device=0)
    for k, v in opts:
        cg.set_option(k, int(v))
    groups.append(cg)
Bh = np.ascontiguousarray(problems.rhs_block(arr)[[0] * R])
dB = torch.from_numpy(Bh).cuda()
dX = torch.zeros_like(dB)
kc = hg.KrylovConfig(restart=10, max_iters=105, rel_tol=1e-12)
streams = [torch.cuda.ExternalStream(cg.stream) for cg in groups]
flush = torch.empty(128 * 1024 * 1024, dtype=torch.float32, device="cuda")


def step():
    e0 = torch.cuda.Event(enable_timing=True)
    e0.record(streams[0])
    for st in streams[1:]:
        st.wait_event(e0)
    th = [threading.Thread(target=lambda g=g: groups[g].fgmres_device(
        "v", dB[bounds[g]:bounds[g + 1]].data_ptr(), dX[bounds[g]:bounds[g + 1]].data_ptr(),
        bounds[g + 1] - bounds[g], kc, want_report=False)) for g in range(G)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    ends = []
    for st in streams:
        e = torch.cuda.Event(enable_timing=True)
        e.record(st)
        ends.append(e)
    torch.cuda.synchronize()
    return max(e0.elapsed_time(e) for e in ends)


base = None
for m in masks:
    for cg in groups:
        cg.set_option("debug_skip", m)
    ts = []
    for k in range(6):
        flush.add_(1.0)
        dX.zero_()
        torch.cuda.synchronize()
        ts.append(step())
    t = float(np.median(ts[2:]))
    rep = groups[0].fgmres_device("v", dB[:4].data_ptr(), dX[:4].data_ptr(), 4, kc, want_report=True)
    if m == 0:
        base = t
    print(f"skip={m:3d}: {t:7.2f} ms/step ({t / 105 * 1e3:6.1f} us/iteration of 444 columns)"
          f"  saved {base - t:6.2f} ms ({(base - t) / base * 100:5.1f}%)  iters={rep.iterations[0]}", flush=True)
