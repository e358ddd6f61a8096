"""Config -> problem arrays from the ORACLE's own generators (TEST
INFRASTRUCTURE: used by tests/, the cpu_baseline leg and the --impl reference
arm of bench.py, so the reference side never loads libhelmgpu.so).

Mirrors paper_2203_11025_b200/problems.py (the product's host plumbing) but
draws the medium (oracle ext A1), the absorbing layer (inc/grid.hpp:98-120)
and the point sources (oracle ext A2) through oracle/liboracle.so.
`tests/test_host_abi.py::test_problem_arrays_product_equals_oracle` pins the
two bit for bit on c0-c4.  Only the config table (plain parameters,
paper_2203_11025_b200/configs.py, no native code) is shared.
"""
from __future__ import annotations

import importlib.util
import os

import numpy as np

from . import oracle as O

_HERE = os.path.dirname(os.path.abspath(__file__))
_CFG_PATH = os.path.join(os.path.dirname(_HERE), "paper_2203_11025_b200", "configs.py")
_configs = None


def configs():
    """The config table, loaded from its file (no package import, no .so)."""
    global _configs
    if _configs is None:
        spec = importlib.util.spec_from_file_location("_hb_configs", _CFG_PATH)
        mod = importlib.util.module_from_spec(spec)
        spec.loader.exec_module(mod)
        _configs = mod
    return _configs


def problem_arrays(cfg: dict) -> dict:
    C = configs()
    n, w = cfg["n"], cfg["abl"]
    om = C.omega_for(n)
    seed, n_if, if_seed = cfg["medium"]
    k2 = O.make_medium(n, n, seed, n_interfaces=n_if, iface_seed=if_seed, margin=w)
    gam = O.absorbing_layer(n, n, w, 2.0 * om)
    xs, ys = C.source_positions(cfg, O.point_sources)
    return dict(n=n, omega=om, kappa2=k2, gamma=gam, lo=C.KAPPA_LO, hi=C.KAPPA_HI, xs=[int(x) for x in xs],
                ys=[int(y) for y in ys])


def rhs_block(arr: dict) -> np.ndarray:
    n = arr["n"]
    B = np.zeros((len(arr["xs"]), n, n), np.complex128)
    for b, (x, y) in enumerate(zip(arr["xs"], arr["ys"])):
        B[b, y, x] = 1.0
    return B
