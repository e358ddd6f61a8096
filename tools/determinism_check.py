import os, sys, numpy as np
sys.path.insert(0, os.getcwd())
import torch
from paper_2203_11025_b200 import helmgpu as hg
g = np.load("tests/golden/train.npz")
CFG = dict(levels=2, base_channels=8, resnet_per_level=1, bottleneck_resnets=1, updown_kernel=5, res_kernel=3)
def garbage():
    x = torch.empty(int(2e9) // 4, device="cuda").fill_(float("nan")); torch.cuda.synchronize(); del x
    torch.cuda.empty_cache()
def pairs():
    ctx = hg.Context(0)
    ctx.set_problem(g["rt_k2"], g["rt_gam"], float(g["rt_om"]), 1/16, 1/2.25)
    ctx.build_hierarchy(hg.VCycleConfig(levels=3))
    r, e, k = ctx.gen_sample_pairs(np.arange(17*6151, 17*6151+5, dtype=np.uint64))
    return r, e, k
def retrain():
    ctx = hg.Context(0)
    ctx.set_paper_net(hg.UNetConfig(**CFG), "standalone")
    ctx.load_checkpoint("tests/golden/train_s_init.unw1")
    ctx.set_problem(g["rt_k2"], g["rt_gam"], float(g["rt_om"]), 1/16, 1/2.25)
    ctx.build_hierarchy(hg.VCycleConfig(levels=3))
    h = ctx.paper_retrain(5, 2, hg.TrainConfig(lr0=1e-3), 17)
    return np.array([e[1] for e in h.epochs]), ctx.paper_param("unet.up1.k")
r1, e1, k1 = pairs(); h1, w1 = retrain()
garbage()
r2, e2, k2 = pairs(); h2, w2 = retrain()
print("k", k1, k2)
print("pairs r diff", np.abs(r1 - r2).max(), "e diff", np.abs(e1 - e2).max(), np.abs(e1).max())
print("hist", h1, h2, "w diff", np.abs(w1 - w2).max())
