import sys, os, numpy as np
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
from test_paper_net import _ctx, GOLD, rel
from paper_2203_11025_b200 import helmgpu as hg
g = np.load(os.path.join(GOLD, "paper.npz"))
n = g["k2"].shape[0]
b = np.zeros((1, n, n), np.complex128); b[0, n // 2, n // 3] = 1.0
for tag in ("s", "es"):
    c = _ctx(hg, g, tag)
    for name, dims in c.paper_params():
        if name.endswith((".b", ".b1", ".b2", ".offset", ".rmean")):
            c.paper_param(name, np.zeros(dims, np.float32))
        if name.endswith("out.k"):
            c.paper_param(name, c.paper_param(name) * np.float32(0.01))
    for kind in ("ju", "vu"):
        print(tag, kind, "z0", rel(c.precond_apply(kind, g["r"]), g[f"{tag}_{kind}_z0"]),
              "small", rel(c.precond_apply(kind, g["r"] * 1e-3), g[f"{tag}_{kind}_zsmall"]),
              "pt", rel(c.precond_apply(kind, b), g[f"{tag}_{kind}_zpt"]))
