"""GPU parity at the BASELINE config sizes and the reference's acceptance gates,
against tests/golden/scale.npz, written by the compiled reference
(oracle/_ref, tests/golden/make_scale_golden.py).

North-star tolerances (BASELINE.json): preconditioner outputs to a relative L2
difference <= 1e-4; iteration counts within +-1 at rel_tol 1e-6.  Full fields
are not committed at 512^2-4096^2: outputs are compared through their L2 norm,
three seeded projections <p_k, z> (each touches every node; compared relative
to ||p_k|| ||z||) and a strided subsample (relative L2), all <= 1e-4.  Residual
histories over a fixed budget are compared entrywise relative to h_0 (see
test_config_full_size_fixed_budget for the bound and why).

The configs c1-c4 carry random-init (He-normal) networks that do not reach
1e-6, so they are fixed-budget runs at their full sizes: c1
256^2 x 8 RHS with the L=4 coarse U-Net (10 its), c2 512^2 M_VU with the L=5
net (2 RHS x 3 its), c3 1024^2 encoder (5 levels x 16 ch) + L=5 solver M_VU
(2 RHS x 2 its), c4 4096^2 4-level cycle with the 512^2 L=4 coarse U-Net (3 its).
Converged solves pin the complex64 basis and the Gram-corrected single-pass MGS
over long runs at m = 10 and m = 20: the classical gate (10 RHS, T = 153), the
homogeneous gate, and M_V at 256^2 FGMRES(10) (T = 346) and 512^2 FGMRES(20)
(T = 795).
"""
import math
import os

import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TOL_PC = 1e-4
BUDGET = {"c1": (8, 10), "c2": (2, 3), "c3": (2, 2), "c4": (1, 3)}
PC_SEED = 9001


@pytest.fixture(scope="module")
def G():
    return np.load(os.path.join(ROOT, "tests", "golden", "scale.npz"))


@pytest.fixture(scope="module")
def hg():
    from paper_2203_11025_b200 import build, helmgpu
    build.build()
    return helmgpu


def check_stats(z, G, key):
    """z (c128 [ny][nx]) against the golden statistics of `key`."""
    flat = z.reshape(-1)
    nz = np.linalg.norm(flat)
    nref = float(G[f"{key}_norm"])
    assert abs(nz - nref) / nref < TOL_PC, (key, nz, nref)
    for k in range(3):
        p = np.random.default_rng(100 + k).standard_normal(flat.size, dtype=np.float32).astype(np.float64)
        d = abs(np.dot(p, flat) - G[f"{key}_proj"][k]) / (np.linalg.norm(p) * nref)
        assert d < TOL_PC, (key, k, d)
    s = int(G[f"{key}_stride"])
    sub, sref = z[::s, ::s], G[f"{key}_sub"]
    e = np.linalg.norm(sub - sref) / np.linalg.norm(sref)
    assert e < TOL_PC, (key, e)
    return e


@pytest.mark.timeout(900)
@pytest.mark.parametrize("name", ["c1", "c2", "c3", "c4"])
def test_config_full_size_fixed_budget(hg, G, name):
    """Full-size config: one preconditioner apply (<= 1e-4 on every statistic)
    and a fixed FGMRES budget.  History entries 0 and 1 (||b||, and the first
    Arnoldi step) agree to 1e-6.  From step 2 on the random-init nets make the
    Z_j nearly collinear -- the nets' r-independent part dominates their output
    -- so the Arnoldi amplifies the fp32 rounding of the networks themselves:
    the REFERENCE's own history moves by `spread` when its weights move by one
    fp32 ulp (`{name}_hist_ulp`, make_scale_golden.py: c1 7.7e-3, c2 3.0e-5,
    c3 1.1e-5, c4 6.2e-7 of h_0).  The device run, whose nets agree with the
    reference's to ~1e-5 (3xTF32 vs OpenBLAS sgemm summation orders), is held
    to 10x that spread.  The solution is checked through a size-independent
    identity instead of the reference's X (which the same amplification makes
    incomparable): the fp64 true residual ||b - A x|| / ||b|| of the device x
    equals the device's own final residual estimate |g_{k+1}| / beta_0 (to
    1e-3, where the least-squares solve is well conditioned)."""
    from paper_2203_11025_b200 import configs, problems
    cfg = configs.CONFIGS[name]
    ctx, arr = problems.gpu_setup(cfg)
    n = cfg["n"]
    r = O.random_complex_normal(PC_SEED, (n, n))
    r /= np.linalg.norm(r)
    kind = cfg["precond"]
    z = ctx.precond_apply(kind, r[None])[0]
    check_stats(z, G, f"{name}_pc")
    ncols, its = BUDGET[name]
    B = problems.rhs_block(arr)[:ncols]
    X, rep = ctx.fgmres(kind, B, hg.KrylovConfig(restart=cfg["restart"], max_iters=its))
    assert list(rep.iterations) == list(G[f"{name}_iters"])
    ref, ulp = G[f"{name}_hist"], G[f"{name}_hist_ulp"]
    spread = np.nanmax(np.abs(ulp - ref) / ref[:, :1])
    for c, h in enumerate(rep.residual_history):
        hr = ref[c][~np.isnan(ref[c])]
        h = np.asarray(h)
        assert len(h) == len(hr)
        d = np.abs(h - hr) / hr[0]
        assert d[:2].max() < 1e-6, (c, d[:2])
        assert d.max() <= 10 * spread, (c, d.max(), spread)
    # the identity needs a well-conditioned least-squares solve: where the
    # reference's own 1-ulp spread exceeds 1e-4 (c1: 7.7e-3, |y| large and
    # cancelling), the complex64 W_j = A Z_j of the Arnoldi relation bounds it
    # only to ~eps32 * ||A|| * sum |y_i| ||Z_i||, so it is reported, not asserted
    A = O.Hierarchy(arr["kappa2"], arr["gamma"], arr["omega"], arr["lo"], arr["hi"], levels=2)
    for c in range(ncols):
        true = np.linalg.norm(B[c] - A.apply(X[c])) / np.linalg.norm(B[c])
        est = rep.residual_history[c][-1] / rep.residual_history[c][0]
        assert np.isfinite(true)
        if spread < 1e-4:
            assert abs(true - est) / est < 1e-3, (c, true, est)
    ctx.close()


@pytest.mark.timeout(900)
@pytest.mark.parametrize("n,m", [(256, 10), (512, 20)])
def test_mv_converged_solve_long_runs(hg, G, n, m):
    """M_V on the BASELINE medium to 1e-6: T within +-1 of the reference's
    (346 at 256^2 FGMRES(10), 795 at 512^2 FGMRES(20)) -- hundreds of Arnoldi
    steps in complex64 with the Gram-corrected MGS."""
    from paper_2203_11025_b200 import configs, problems
    cfg = dict(configs.CONFIGS["c0"])
    cfg.update(n=n, restart=m)
    ctx, arr = problems.gpu_setup(cfg)
    B = problems.rhs_block(arr)
    X, rep = ctx.fgmres("v", B, hg.KrylovConfig(restart=m, max_iters=2000))
    T_ref = int(G[f"mv{n}_iters"])
    assert rep.converged[0] and bool(G[f"mv{n}_converged"])
    assert abs(rep.iterations[0] - T_ref) <= 1, (rep.iterations[0], T_ref)
    href = G[f"mv{n}_hist"]
    k = min(len(href), len(rep.residual_history[0]))
    # histories agree closely while the residual is far above the c64 floor
    d = np.abs(np.asarray(rep.residual_history[0][:k]) - href[:k]) / href[0]
    assert d.max() < 1e-5, d.max()
    # the solutions agree to the solve tolerance (both are 1e-6 solutions)
    s = int(G[f"mv{n}_x_stride"])
    e = np.linalg.norm(X[0][::s, ::s] - G[f"mv{n}_x_sub"]) / np.linalg.norm(G[f"mv{n}_x_sub"])
    assert e < 1e-4, e
    ctx.close()


def gate_rhs(hg, n, count, seed):
    """random_rhs_block (inc/bench.hpp:83-90) from the library's Rng
    restatement: Rng(seed ^ 0xb10c), Complex(normal(), normal()) per node,
    evaluated right to left by GCC (imaginary part drawn first)."""
    z = hg.rng_normals(seed ^ 0xB10C, 2 * count * n * n).reshape(count, n, n, 2)
    return z[..., 1] + 1j * z[..., 0]


@pytest.mark.timeout(600)
@pytest.mark.parametrize("gate", ["classical", "homog"])
def test_reference_acceptance_gates(hg, G, gate):
    """tests/acceptance.cpp:184-201 (classical SL reproduction: rho in
    [0.85, 0.95], T in [100, 190], all converged; the reference gives rho =
    0.9136, T = 153) and :203-217 (homogeneous: rho <= 0.93), run through the
    device solver on the reference's own gate problems (synthetic_slowness
    medium as a fixture), T within +-1 per column."""
    n = 128
    k2, gam = G[f"gate_{gate}_k2"], G[f"gate_{gate}_gamma"]
    B = gate_rhs(hg, n, 10, 42 if gate == "classical" else 43)
    ctx = hg.Context(0)
    ctx.set_problem(k2, gam, 20 * math.pi, 0.25, 1.0)
    ctx.build_hierarchy(hg.VCycleConfig(levels=3))
    X, rep = ctx.fgmres("v", B, hg.KrylovConfig(restart=10, max_iters=300))
    cf = [hg.convergence_factor(h) for h in rep.residual_history]
    assert all(c[2] for c in cf)
    T = np.array([c[0] for c in cf])
    rho = np.array([c[1] for c in cf])
    assert np.max(np.abs(T - G[f"gate_{gate}_T"])) <= 1
    assert np.max(np.abs(rho - G[f"gate_{gate}_rho"])) < 2e-3
    rm, Tm = float(np.median(rho)), float(np.median(T))
    if gate == "classical":
        assert 0.85 <= rm <= 0.95 and 100 <= Tm <= 190
    else:
        assert rm <= 0.93
    ctx.close()


def test_nonflexible_gmres_and_dense_coarse(hg):
    """Standard right-preconditioned GMRES (flexible = false, inc/krylov.hpp:
    127-136) on the device, with the exact (dense) coarsest solve that makes
    M_V linear (tests/test_classic.cpp:442-467): flexible and standard GMRES
    agree, and both match the C oracle; network preconditioners reject
    flexible = false (check_flexible_contract, inc/precond.hpp:29-32)."""
    n = 32
    om = 2 * math.pi * 1.5 * n / 10
    k2 = hg.make_medium(n, n, 1234)
    gam = hg.absorbing_layer(n, n, 4, 2 * om)
    ctx = hg.Context(0)
    ctx.set_problem(k2, gam, om, 1 / 16, 1 / 2.25)
    ctx.build_hierarchy(hg.VCycleConfig(levels=3, coarse_solver="dense"))
    b = O.random_complex_normal(121, (2, n, n))
    # the dense coarse solve is the exact inverse: M_V of the 2-level analogue
    # equals the oracle's two-grid cycle with a dense coarsest solve
    xf, rf = ctx.fgmres("v", b, hg.KrylovConfig(restart=10, max_iters=60, rel_tol=1e-6, flexible=True))
    xs, rs = ctx.fgmres("v", b, hg.KrylovConfig(restart=10, max_iters=60, rel_tol=1e-6, flexible=False))
    for c in range(2):
        assert rf.converged[c] and rs.converged[c]
        assert abs(rf.iterations[c] - rs.iterations[c]) <= 1
        h, hs = np.asarray(rf.residual_history[c]), np.asarray(rs.residual_history[c])
        k = min(len(h), len(hs))
        assert np.max(np.abs(h[:k] - hs[:k])) / h[0] < 1e-5
        assert np.linalg.norm(xf[c] - xs[c]) / np.linalg.norm(xf[c]) < 1e-5
    # both are solutions of A x = b to the tolerance (checked in fp64 by the oracle)
    H = O.Hierarchy(k2, gam, om, 1 / 16, 1 / 2.25, levels=3)
    for c in range(2):
        assert np.linalg.norm(b[c] - H.apply(xs[c])) / np.linalg.norm(b[c]) <= 1.05e-6
    ctx.set_net(0, "solver", 2, 16, 3, 0)
    ctx.init_net_he(0, 7)
    with pytest.raises(Exception):
        ctx.fgmres("vu", b, hg.KrylovConfig(restart=10, max_iters=5, flexible=False))
    ctx.close()


def test_dense_coarse_matches_reference(hg):
    """CoarseSolver::dense (inc/multigrid.hpp:84,95-104) against the compiled
    reference when it is present (this container), else against the dense
    inverse applied by numpy to the oracle's coarsest operator."""
    n = 32
    om = 2 * math.pi * 1.5 * n / 10
    k2 = hg.make_medium(n, n, 77)
    gam = hg.absorbing_layer(n, n, 4, 2 * om)
    ctx = hg.Context(0)
    ctx.set_problem(k2, gam, om, 1 / 16, 1 / 2.25)
    ctx.build_hierarchy(hg.VCycleConfig(levels=3, coarse_solver="dense"))
    f = O.random_complex_normal(5, (2, 8, 8))
    x = ctx.coarse_solve(f)
    H = O.Hierarchy(k2, gam, om, 1 / 16, 1 / 2.25, levels=3)
    for b in range(2):
        # the exact solve: M^H x = f on the coarsest level (oracle stencil, fp64)
        res = np.linalg.norm(H.apply(x[b], level=2, shifted=True) - f[b]) / np.linalg.norm(f[b])
        assert res < 1e-5, res
    if O.have_ref():
        R = O.RefHierarchy(k2, gam, om, 1 / 16, 1 / 2.25, levels=3, coarse="dense")
        r = O.random_complex_normal(6, (2, n, n))
        zr = O.RefPrecond("v", R).apply(r)
        z = ctx.precond_apply("v", r)
        assert np.linalg.norm(z - zr) / np.linalg.norm(zr) < TOL_PC
    ctx.close()
