"""B200-native (sm_100a) hot path of arXiv 2203.11025: FGMRES on the 2-D
Helmholtz operator preconditioned by a shifted-Laplacian V-cycle combined with
a U-Net.  The compute lives in libhelmgpu.so (CUDA, C ABI in
include/helmgpu.h); this package is the Python host mirror of the reference's
solver / preconditioner API used by tests and bench.py."""
from .configs import CONFIGS, omega_for  # noqa: F401

__all__ = ["CONFIGS", "omega_for"]
