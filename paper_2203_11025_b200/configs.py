"""The five BASELINE.json configurations (plus their literal variants), as
plain parameters.  SURVEY.md 8(d) "Synthetic inputs" and Appendix A fix the
seeds and the decisions D0-D10 that these encode.

omega = 2*pi*1.5*n/10 puts 10 points per wavelength at the minimum velocity
1.5 (inc/grid.hpp:138 bound omega*kappa*h <= 0.6284 holds with equality to
1e-5); gamma_max = 2*omega (D2); kappa^2 = 1/c^2 declared on [1/16, 1/2.25].
"""
from __future__ import annotations

import math

KAPPA_LO = 1.0 / 16.0
KAPPA_HI = 1.0 / 2.25


def omega_for(n: int) -> float:
    return 2.0 * math.pi * 1.5 * n / 10.0


# net: (levels, base channels, He seed, context channels); enc: (levels, base, seed)
CONFIGS = {
    # c0: M_V, 3 levels, reference GMRES(10) coarsest (headline variant, D1)
    "c0": dict(n=128, abl=16, levels=3, coarse="gmres", coarse_iters=10, restart=10, B=1,
               sources=("center",), medium=(1234, 0, 0), precond="v", net=None, enc=None, max_iters=2000),
    # c0 literal: 20 damped-Jacobi sweeps on the coarsest grid (A3; does not converge)
    "c0j": dict(n=128, abl=16, levels=3, coarse="jacobi", coarse_iters=20, restart=10, B=1,
                sources=("center",), medium=(1234, 0, 0), precond="v", net=None, enc=None, max_iters=200),
    # c1: 2-level SL cycle with the classic U-Net (L=4, 16..128) as coarse solver (A4)
    "c1": dict(n=256, abl=16, levels=2, coarse="net", coarse_iters=0, restart=10, B=8,
               sources=("uniform", 42), medium=(1234, 0, 0), precond="v", net=(4, 16, 7, 0), enc=None,
               max_iters=200),
    # c2: M_VU (A8), U-Net L=5 (16..256) at 512^2 + 3-level V-cycle, medium with 3 interfaces (D7)
    "c2": dict(n=512, abl=16, levels=3, coarse="gmres", coarse_iters=10, restart=20, B=16,
               sources=("uniform", 43), medium=(1234, 3, 1235), precond="vu", net=(5, 16, 8, 0), enc=None,
               max_iters=200),
    "c2j": dict(n=512, abl=16, levels=3, coarse="jacobi", coarse_iters=20, restart=20, B=16,
                sources=("uniform", 43), medium=(1234, 3, 1235), precond="vu", net=(5, 16, 8, 0), enc=None,
                max_iters=200),
    # c3: encoder-solver M_VU (A7), 64 sources on row abl+4
    "c3": dict(n=1024, abl=16, levels=3, coarse="gmres", coarse_iters=10, restart=20, B=64,
               sources=("row", 44), medium=(1234, 0, 0), precond="vu", net=(5, 16, 9, 16), enc=(5, 16, 10),
               max_iters=200),
    # c4: single 4096^2 problem, 4-level V-cycle, U-Net (L=4) coarse solver at 512^2
    "c4": dict(n=4096, abl=32, levels=4, coarse="net", coarse_iters=0, restart=20, B=1,
               sources=("center",), medium=(1234, 0, 0), precond="v", net=(4, 16, 11, 0), enc=None,
               max_iters=200),
}


def source_positions(cfg, point_sources_fn):
    """(xs, ys) of the unit point sources (oracle ext A2).  point_sources_fn is
    the seeded generator (GPU host library or oracle; both restate Rng)."""
    n, w, B = cfg["n"], cfg["abl"], cfg["B"]
    kind = cfg["sources"][0]
    if kind == "center":
        return [n // 2] * B, [n // 2] * B
    if kind == "uniform":
        return point_sources_fn(cfg["sources"][1], B, 0, w, n - w - 1, 0)
    if kind == "row":
        return point_sources_fn(cfg["sources"][1], B, 1, w, n - w - 1, w + 4)
    raise ValueError(kind)


def scaled(cfg_name: str, n: int, B: int | None = None) -> dict:
    """A config with the same structure at a smaller grid (parity tests)."""
    c = dict(CONFIGS[cfg_name])
    c["n"] = n
    c["abl"] = max(2, min(c["abl"], n // 8))
    if B is not None:
        c["B"] = B
    return c
