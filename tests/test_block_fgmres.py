"""True block FGMRES (hb_block_fgmres): all right-hand
sides share one block Krylov space.  Checked against the fp64 numpy
restatement of the published algorithm (oracle.block_fgmres_np, with the C
oracle's M_V and stencil as operators), against the column-wise device
FGMRES at block size 1, and through the residual contract in fp64."""
import math

import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def hg():
    from paper_2203_11025_b200 import build, helmgpu
    build.build()
    return helmgpu


def setup(hg, n=64, abl=8):
    om = 2 * math.pi * 1.5 * n / 10
    k2 = hg.make_medium(n, n, 1234)
    g = hg.absorbing_layer(n, n, abl, 2 * om)
    ctx = hg.Context(0)
    ctx.set_problem(k2, g, om, 1 / 16, 1 / 2.25)
    ctx.build_hierarchy(hg.VCycleConfig(levels=3))
    H = O.Hierarchy(k2, g, om, 1 / 16, 1 / 2.25, levels=3)
    return ctx, H


def test_block_size_one_equals_fgmres(hg):
    ctx, _ = setup(hg)
    b = O.random_complex_normal(5, (1, 64, 64))
    cfg = hg.KrylovConfig(restart=10, max_iters=200)
    Xb, rb = ctx.block_fgmres("v", b, cfg)
    Xs, rs = ctx.fgmres("v", b, cfg)
    assert rb.converged[0] and rs.converged[0]
    assert abs(rb.iterations[0] - rs.iterations[0]) <= 1
    hb, hs = np.asarray(rb.residual_history[0]), np.asarray(rs.residual_history[0])
    k = min(len(hb), len(hs))
    assert np.max(np.abs(hb[:k] - hs[:k])) / hs[0] < 1e-5
    assert np.linalg.norm(Xb - Xs) / np.linalg.norm(Xs) < 1e-4


@pytest.mark.parametrize("p", [3, 8])
def test_block_fgmres_matches_numpy_oracle(hg, p):
    ctx, H = setup(hg)
    B = O.random_complex_normal(100 + p, (p, 64, 64))
    cfg = hg.KrylovConfig(restart=8, max_iters=120, rel_tol=1e-6)
    X, rep = ctx.block_fgmres("v", B, cfg)
    P = O.Precond("v", H)
    apply_A = lambda U: np.stack([H.apply(u) for u in U])  # noqa: E731
    Xo, ho, ito = O.block_fgmres_np(apply_A, P.apply, B, restart=8, max_iters=120, rel_tol=1e-6)
    assert all(rep.converged)
    assert abs(rep.iterations[0] - ito) <= 1, (rep.iterations[0], ito)
    for c in range(p):
        h, hr = np.asarray(rep.residual_history[c]), ho[c]
        k = min(len(h), len(hr))
        # the histories agree while the residual is far above the c64 floor
        assert np.max(np.abs(h[:k] - hr[:k])) / hr[0] < 1e-4, c
        res = np.linalg.norm(B[c] - H.apply(X[c])) / np.linalg.norm(B[c])
        assert res <= 1.05e-6, (c, res)
    assert np.linalg.norm(X - Xo) / np.linalg.norm(Xo) < 1e-4
    # one shared Krylov space: no more block steps than the column-wise solve needs
    Xs, rs = ctx.fgmres("v", B, hg.KrylovConfig(restart=8, max_iters=400))
    assert rep.iterations[0] <= max(rs.iterations)


def test_block_fgmres_rejects_bad_config(hg):
    ctx, _ = setup(hg)
    B = O.random_complex_normal(1, (2, 64, 64))
    with pytest.raises(Exception):
        ctx.block_fgmres("v", B, hg.KrylovConfig(restart=10, max_iters=20, flexible=False))
    with pytest.raises(Exception):
        ctx.block_fgmres("v", np.zeros((17, 64, 64)), hg.KrylovConfig(restart=10, max_iters=20))
    X, rep = ctx.block_fgmres("v", np.zeros((2, 64, 64)), hg.KrylovConfig(restart=10, max_iters=20))
    assert np.all(X == 0) and all(rep.converged)
