"""Config -> problem/hierarchy/net setup on the GPU library (host plumbing for
tests and bench.py).  Inputs are the seeded synthetic media and point sources
of SURVEY.md 8(d); the generators are the library's own host restatements."""
from __future__ import annotations

import numpy as np

from . import helmgpu as hg
from .configs import CONFIGS, KAPPA_HI, KAPPA_LO, omega_for, source_positions


def problem_arrays(cfg: dict):
    n, w = cfg["n"], cfg["abl"]
    om = omega_for(n)
    seed, n_if, if_seed = cfg["medium"]
    k2 = hg.make_medium(n, n, seed, n_interfaces=n_if, iface_seed=if_seed, margin=w)
    gam = hg.absorbing_layer(n, n, w, 2.0 * om)
    xs, ys = source_positions(cfg, hg.point_sources)
    return dict(n=n, omega=om, kappa2=k2, gamma=gam, lo=KAPPA_LO, hi=KAPPA_HI, xs=list(xs), ys=list(ys))


def rhs_block(arr: dict) -> np.ndarray:
    n = arr["n"]
    B = np.zeros((len(arr["xs"]), n, n), np.complex128)
    for b, (x, y) in enumerate(zip(arr["xs"], arr["ys"])):
        B[b, y, x] = 1.0
    return B


def vcycle_config(cfg: dict) -> hg.VCycleConfig:
    return hg.VCycleConfig(levels=cfg["levels"], nu1=1, nu2=1, damping=0.8, alpha=1.0, beta=0.5,
                           coarse_iters=max(1, cfg["coarse_iters"]) if cfg["coarse"] != "net" else 1,
                           coarse_solver=cfg["coarse"])


def gpu_setup(cfg: dict, device: int = 0, arr: dict | None = None) -> tuple[hg.Context, dict]:
    arr = arr or problem_arrays(cfg)
    ctx = hg.Context(device)
    ctx.set_problem(arr["kappa2"], arr["gamma"], arr["omega"], arr["lo"], arr["hi"])
    ctx.build_hierarchy(vcycle_config(cfg))
    if cfg["net"] is not None:
        L, base, seed, ctx_ch = cfg["net"]
        ctx.set_net(0, "solver", L, base, 3, ctx_ch)
        ctx.init_net_he(0, seed)
    if cfg["enc"] is not None:
        L, base, seed = cfg["enc"]
        ctx.set_net(1, "encoder", L, base, 1, 0)
        ctx.init_net_he(1, seed)
        ctx.encode()
    return ctx, arr


def get(name: str) -> dict:
    return dict(CONFIGS[name])
