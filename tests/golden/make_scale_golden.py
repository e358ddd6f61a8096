"""Generate tests/golden/scale.npz from the REFERENCE ITSELF (oracle/_ref: the
unmodified reference headers compiled in place by oracle/build_ref.sh) at the
BASELINE config sizes, plus the reference's own acceptance gates.  Run here
(where /root/reference exists); the fixture is committed so the GPU box checks
against it without the reference.

    bash oracle/build_ref.sh && python tests/golden/make_scale_golden.py [--only NAME,...]

Contents (c128 fields are too large to commit at 512^2-4096^2, so every
preconditioner output is summarised by size-independent statistics that touch
every node: its L2 norm, K = 3 projections <p_k, z> on seeded fp32 weight
fields p_k ~ N(0, 1) (np.random.default_rng(100 + k)), and a strided
subsample z[::s, ::s] of at most 128 x 128 nodes):

  gate_classical_*   tests/acceptance.cpp:184-201: 128^2, omega = 20 pi,
                     synthetic_slowness(5 * 1000003), ABL 10 / 0.5, M_V,
                     block FGMRES(10) of random_rhs_block(10, seed 42), 300 its
  gate_homog_*       tests/acceptance.cpp:203-217: kappa^2 = 1, rhs seed 43
  mv256_* / mv512_*  converged M_V solves on the BASELINE medium (centre point
                     source): 256^2 FGMRES(10), 512^2 FGMRES(20) (SURVEY App. B:
                     T = 346 / 795)
  c1_* .. c4_*       fixed-budget FGMRES on the BASELINE configs at full size
                     (c1: 8 RHS x 10 its; c2: 2 RHS x 3; c3: 2 RHS x 2; c4: 1 x 3)
                     and one preconditioner apply on a seeded complex-normal r
"""
from __future__ import annotations

import math
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle import oracle as O  # noqa: E402
from oracle import problems as OP  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "scale.npz")

# fixed budgets: (columns, FGMRES iterations)
BUDGET = {"c1": (8, 10), "c2": (2, 3), "c3": (2, 2), "c4": (1, 3)}
PC_SEED = 9001  # seed of the complex-normal preconditioner input


def field_stats(z):
    """(norm, projections[3], subsample, stride) of a c128 field [ny][nx]."""
    ny, nx = z.shape
    flat = z.reshape(-1)
    proj = []
    for k in range(3):
        p = np.random.default_rng(100 + k).standard_normal(flat.size, dtype=np.float32)
        proj.append(np.dot(p.astype(np.float64), flat))
    s = max(1, nx // 128)
    return float(np.linalg.norm(flat)), np.array(proj), np.ascontiguousarray(z[::s, ::s]), s


def pack_hist(hists):
    L = max(len(h) for h in hists)
    out = np.full((len(hists), L), np.nan)
    for i, h in enumerate(hists):
        out[i, :len(h)] = h
    return out


def gates(g):
    def convergence_factor(h):  # inc/bench.hpp:22-38 via the oracle's restatement
        T, rho = O.convergence_factor(np.asarray(h))
        return abs(T), rho

    n = 128
    om = 20 * math.pi
    gam = np.zeros((n, n))
    O.ref().hr_absorbing_layer(n, n, 10, 0.5, O._p(gam))
    for name, k2, seed in (("classical", O.ref_synthetic_slowness(5 * 1000003, n, n), 42),
                           ("homog", np.ones((n, n)), 43)):
        B = O.ref_random_rhs_block(n, n, 10, seed)
        H = O.RefHierarchy(k2, gam, om, 0.25, 1.0, levels=3)
        P = O.RefPrecond("v", H)
        t0 = time.time()
        X, rep = O.ref_fgmres(P, B, restart=10, max_iters=300, nthreads=10)
        cf = [convergence_factor(h) for h in rep["history"]]
        g[f"gate_{name}_k2"] = k2
        g[f"gate_{name}_gamma"] = gam
        g[f"gate_{name}_hist"] = pack_hist(rep["history"])
        g[f"gate_{name}_T"] = np.array([c[0] for c in cf])
        g[f"gate_{name}_rho"] = np.array([c[1] for c in cf])
        print(f"gate {name}: T median {np.median(g[f'gate_{name}_T'])}, rho median "
              f"{np.median(g[f'gate_{name}_rho']):.4f} ({time.time() - t0:.1f} s)", flush=True)


def mv_solves(g):
    for n, m in ((256, 10), (512, 20)):
        cfg = dict(OP.configs().CONFIGS["c0"])
        cfg.update(n=n, restart=m)
        arr = OP.problem_arrays(cfg)
        B = OP.rhs_block(arr)
        H = O.RefHierarchy(arr["kappa2"], arr["gamma"], arr["omega"], arr["lo"], arr["hi"], levels=3)
        P = O.RefPrecond("v", H)
        t0 = time.time()
        X, rep = O.ref_fgmres(P, B, restart=m, max_iters=2000)
        g[f"mv{n}_hist"] = rep["history"][0]
        g[f"mv{n}_iters"] = int(rep["iterations"][0])
        g[f"mv{n}_converged"] = bool(rep["converged"][0])
        xs = field_stats(X[0])
        g[f"mv{n}_x_norm"], g[f"mv{n}_x_proj"], g[f"mv{n}_x_sub"], g[f"mv{n}_x_stride"] = xs
        print(f"M_V {n}^2 FGMRES({m}): T = {rep['iterations'][0]} converged {rep['converged'][0]} "
              f"({time.time() - t0:.1f} s)", flush=True)


def configs(g, names):
    import bench  # ref_preconditioner: the reference's preconditioner for a config
    for name in names:
        cfg = dict(OP.configs().CONFIGS[name])
        arr = OP.problem_arrays(cfg)
        ncols, its = BUDGET[name]
        t0 = time.time()
        H, P = bench.ref_preconditioner(O, "reference", cfg, arr)
        n = cfg["n"]
        r = O.random_complex_normal(PC_SEED, (n, n))
        r /= np.linalg.norm(r)
        z = P.apply(r)[0]
        st = field_stats(z)
        g[f"{name}_pc_norm"], g[f"{name}_pc_proj"], g[f"{name}_pc_sub"], g[f"{name}_pc_stride"] = st
        t1 = time.time()
        B = OP.rhs_block(arr)[:ncols]
        X, rep = O.ref_fgmres(P, B, restart=cfg["restart"], max_iters=its, nthreads=ncols)
        g[f"{name}_hist"] = pack_hist(rep["history"])
        g[f"{name}_iters"] = np.array(rep["iterations"])
        xs = field_stats(X[0])
        g[f"{name}_x_norm"], g[f"{name}_x_proj"], g[f"{name}_x_sub"], g[f"{name}_x_stride"] = xs
        # the reference's own sensitivity: the same solve with every network weight
        # moved by ~1 fp32 ulp (x (1 + 2^-22)).  The random-init nets make the Z_j
        # nearly collinear (their r-independent part dominates), so the Arnoldi from
        # step 2 on amplifies fp32 rounding of the net; a device run is held to a
        # small multiple of this spread (tests/test_scale_parity.py)
        for net in P._keep[:2]:
            if net is not None:
                for w, bias in net.convs():
                    w *= np.float32(1.0 + 2.0 ** -22)
        X2, rep2 = O.ref_fgmres(P, B, restart=cfg["restart"], max_iters=its, nthreads=ncols)
        g[f"{name}_hist_ulp"] = pack_hist(rep2["history"])
        spread = np.nanmax(np.abs(g[f"{name}_hist_ulp"] - g[f"{name}_hist"]) / g[f"{name}_hist"][:, :1])
        print(f"{name}: apply {t1 - t0:.1f} s, {ncols} x {its} FGMRES its {time.time() - t1:.1f} s, "
              f"rel residual end {[round(float(h[-1] / h[0]), 6) for h in rep['history']]}, "
              f"1-ulp history spread {spread:.3e}", flush=True)
        del P, H


def main():
    only = None
    if "--only" in sys.argv:
        only = sys.argv[sys.argv.index("--only") + 1].split(",")
    g = dict(np.load(OUT)) if (only and os.path.exists(OUT)) else {}
    if not only or "gates" in only:
        gates(g)
    if not only or "mv" in only:
        mv_solves(g)
    names = [c for c in ("c1", "c2", "c3", "c4") if not only or c in only]
    configs(g, names)
    np.savez_compressed(OUT, **g)
    print("wrote", OUT, os.path.getsize(OUT), "bytes")


if __name__ == "__main__":
    main()
