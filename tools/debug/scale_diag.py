"""Diagnostic: per-config deviation of the device fixed-budget runs from the
reference goldens (tests/golden/scale.npz): preconditioner stats, history
deviations per iteration, solution stats."""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle import oracle as O  # noqa: E402
from paper_2203_11025_b200 import configs, helmgpu as hg, problems  # noqa: E402

G = np.load(os.path.join(ROOT, "tests", "golden", "scale.npz"))
BUDGET = {"c1": (8, 10), "c2": (2, 3), "c3": (2, 2), "c4": (1, 3)}


def stats_err(z, key):
    flat = z.reshape(-1)
    nref = float(G[f"{key}_norm"])
    out = {"norm": abs(np.linalg.norm(flat) - nref) / nref}
    pe = []
    for k in range(3):
        p = np.random.default_rng(100 + k).standard_normal(flat.size, dtype=np.float32).astype(np.float64)
        pe.append(abs(np.dot(p, flat) - G[f"{key}_proj"][k]) / (np.linalg.norm(p) * nref))
    out["proj"] = max(pe)
    s = int(G[f"{key}_stride"])
    out["sub"] = float(np.linalg.norm(z[::s, ::s] - G[f"{key}_sub"]) / np.linalg.norm(G[f"{key}_sub"]))
    return out


for name in sys.argv[1:] or ["c1", "c2", "c3", "c4"]:
    cfg = configs.CONFIGS[name]
    ctx, arr = problems.gpu_setup(cfg)
    n = cfg["n"]
    r = O.random_complex_normal(9001, (n, n))
    r /= np.linalg.norm(r)
    z = ctx.precond_apply(cfg["precond"], r[None])[0]
    res = {"config": name, "pc": stats_err(z, f"{name}_pc")}
    nc, its = BUDGET[name]
    B = problems.rhs_block(arr)[:nc]
    X, rep = ctx.fgmres(cfg["precond"], B, hg.KrylovConfig(restart=cfg["restart"], max_iters=its))
    dev = []
    for c in range(nc):
        hr = G[f"{name}_hist"][c]
        hr = hr[~np.isnan(hr)]
        h = np.asarray(rep.residual_history[c])
        dev.append([float(x) for x in np.abs(h[:len(hr)] - hr[:len(h)]) / hr[0]])
    res["hist_dev"] = dev
    res["x"] = stats_err(X[0], f"{name}_x")
    print(json.dumps(res), flush=True)
    ctx.close()
