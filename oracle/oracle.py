"""ctypes wrapper over the CPU oracle (oracle/liboracle.so) and the compiled
reference (oracle/_ref/libhelmref.so).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and the
cpu_baseline / --impl reference legs of bench.py.  The GPU product
(paper_2203_11025_b200) never imports this module.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liboracle.so")
REF_PATH = os.path.join(HERE, "_ref", "libhelmref.so")

_dp = C.POINTER(C.c_double)
_fp = C.POINTER(C.c_float)
_ip = C.POINTER(C.c_int)
_vp = C.c_void_p


def build(force: bool = False) -> str:
    """Compile the C restatement (gcc, -O3, OpenMP over independent columns)."""
    src = os.path.join(HERE, "helm_oracle.c")
    if force or not os.path.exists(LIB_PATH) or os.path.getmtime(LIB_PATH) < os.path.getmtime(src):
        subprocess.check_call(["gcc", "-O3", "-fPIC", "-shared", "-fopenmp", "-o", LIB_PATH, src, "-lm"])
    return LIB_PATH


def _p(a, t=_dp):
    return a.ctypes.data_as(t) if a is not None else None


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        L = C.CDLL(LIB_PATH)
        L.ho_unet_create.restype = _vp
        L.ho_unet_create.argtypes = [C.c_int] * 5
        L.ho_unet_conv_weight.restype = _fp
        L.ho_unet_conv_weight.argtypes = [_vp, C.c_int]
        L.ho_unet_conv_bias.restype = _fp
        L.ho_unet_conv_bias.argtypes = [_vp, C.c_int]
        L.ho_unet_nconv.argtypes = [_vp]
        L.ho_unet_conv_shape.argtypes = [_vp, C.c_int, _ip, _ip]
        L.ho_unet_init_he.argtypes = [_vp, C.c_uint64]
        L.ho_unet_destroy.argtypes = [_vp]
        L.ho_unet_forward.argtypes = [_vp, C.c_int, C.c_int, C.c_int, _fp, C.POINTER(_fp), _fp]
        L.ho_encoder_forward.argtypes = [_vp, C.c_int, C.c_int, _fp, C.POINTER(_fp)]
        L.ho_mg_create.restype = _vp
        L.ho_mg_create.argtypes = [C.c_int, C.c_int, C.c_double, C.c_double, _dp, _dp, C.c_double, C.c_double,
                                   C.c_int, C.c_int, C.c_int, C.c_double, C.c_double, C.c_double, C.c_int,
                                   C.c_int]
        L.ho_mg_destroy.argtypes = [_vp]
        L.ho_mg_set_coarse_net.argtypes = [_vp, _vp]
        L.ho_mg_level_info.argtypes = [_vp, C.c_int, _ip, _ip, _dp]
        L.ho_mg_level_coef.argtypes = [_vp, C.c_int, _dp, _dp, _dp, _dp]
        L.ho_apply.argtypes = [_vp, C.c_int, C.c_int, _dp, _dp]
        L.ho_jacobi.argtypes = [_vp, C.c_int, C.c_int, _dp, _dp, C.c_double, C.c_int]
        L.ho_mg_cycle.argtypes = [_vp, _dp, _dp, _dp]
        L.ho_coarse_gmres.argtypes = [_vp, C.c_int, C.c_int, _dp, _dp]
        L.ho_pc_create.restype = _vp
        L.ho_pc_create.argtypes = [C.c_int, _vp, _vp, _vp]
        L.ho_pc_destroy.argtypes = [_vp]
        L.ho_pc_apply.argtypes = [_vp, C.c_int, _dp, _dp]
        L.ho_pc_net_guess.argtypes = [_vp, _dp, _dp]
        L.ho_pc_ctx.restype = _fp
        L.ho_pc_ctx.argtypes = [_vp, C.c_int]
        L.ho_fgmres.argtypes = [_vp, C.c_int, C.c_int, C.c_double, C.c_int, C.c_int, _dp, _dp, _dp, C.c_int,
                                _ip, _ip, _ip, _ip, C.c_int]
        L.ho_restrict.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, _dp, _dp]
        L.ho_prolong.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, _dp, _dp]
        L.ho_absorbing_layer.argtypes = [C.c_int, C.c_int, C.c_int, C.c_double, _dp]
        L.ho_make_medium.argtypes = [C.c_int, C.c_int, C.c_uint64, C.c_double, C.c_double, C.c_double, C.c_int,
                                     C.c_uint64, C.c_int, C.c_double, C.c_double, _dp]
        L.ho_point_sources.argtypes = [C.c_uint64, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, _ip, _ip]
        L.ho_rng_normals.argtypes = [C.c_uint64, C.c_int64, _dp]
        L.ho_random_complex_normal.argtypes = [C.c_uint64, C.c_int64, _dp]
        L.ho_gaussian_blur.argtypes = [C.c_int, C.c_int, C.c_double, _dp, _dp]
        L.ho_op_conv3x3.argtypes = [C.c_int] * 5 + [_fp, _fp, _fp, C.c_int, _fp]
        L.ho_op_maxpool2.argtypes = [C.c_int] * 4 + [_fp, _fp]
        L.ho_op_upsample2.argtypes = [C.c_int] * 4 + [_fp, _fp]
        L.ho_convergence_factor.argtypes = [_dp, C.c_int, C.c_double, _dp]
        _lib = L
    return _lib


# ----------------------------------------------------------------- helpers
def cfield(a):
    """complex128 array -> contiguous complex128 (viewed as interleaved doubles)"""
    return np.ascontiguousarray(a, dtype=np.complex128)


def cptr(a):
    return a.ctypes.data_as(_dp)


def absorbing_layer(nx, ny, width, gmax):
    out = np.zeros((ny, nx))
    if lib().ho_absorbing_layer(nx, ny, width, gmax, _p(out)) != 0:
        raise ValueError("absorbing layer width / gamma_max out of range")
    return out


def make_medium(nx, ny, seed, sigma=8.0, vmin=1.5, vmax=4.0, n_interfaces=0, iface_seed=0, margin=16,
                jmin=0.5, jmax=1.0):
    out = np.zeros((ny, nx))
    lib().ho_make_medium(nx, ny, seed, sigma, vmin, vmax, n_interfaces, iface_seed, margin, jmin, jmax, _p(out))
    return out


def point_sources(seed, B, mode, lo, hi, row=0):
    xs = np.zeros(B, np.int32)
    ys = np.zeros(B, np.int32)
    lib().ho_point_sources(seed, B, mode, lo, hi, row, _p(xs, _ip), _p(ys, _ip))
    return xs, ys


def random_complex_normal(seed, shape):
    n = int(np.prod(shape))
    out = np.zeros(n, np.complex128)
    lib().ho_random_complex_normal(seed, n, cptr(out))
    return out.reshape(shape)


class UNet:
    """Classic U-Net (kind 0) or context encoder (kind 1); oracle ext A5-A7."""

    def __init__(self, kind, L, base, in_ch, ctx_ch=0, seed=None):
        self.kind, self.L, self.base, self.in_ch, self.ctx_ch = kind, L, base, in_ch, ctx_ch
        self.h = lib().ho_unet_create(kind, L, base, in_ch, ctx_ch)
        if not self.h:
            raise ValueError("bad U-Net config")
        if seed is not None:
            lib().ho_unet_init_he(self.h, seed)

    def __del__(self):
        if getattr(self, "h", None):
            lib().ho_unet_destroy(self.h)
            self.h = None

    def convs(self):
        """list of (weight view (cout,cin,3,3), bias view (cout,)) in creation order"""
        out = []
        for i in range(lib().ho_unet_nconv(self.h)):
            co, ci = C.c_int(), C.c_int()
            lib().ho_unet_conv_shape(self.h, i, C.byref(co), C.byref(ci))
            w = np.ctypeslib.as_array(lib().ho_unet_conv_weight(self.h, i), shape=(co.value, ci.value, 3, 3))
            b = np.ctypeslib.as_array(lib().ho_unet_conv_bias(self.h, i), shape=(co.value,))
            out.append((w, b))
        return out

    def forward(self, x, ctx=None):
        x = np.ascontiguousarray(x, np.float32)
        B, _, H, W = x.shape
        out = np.zeros((B, 2, H, W), np.float32)
        cp = None
        if ctx is not None:
            ctx = [np.ascontiguousarray(c, np.float32) for c in ctx]
            cp = (_fp * len(ctx))(*[_p(c, _fp) for c in ctx])
        lib().ho_unet_forward(self.h, B, H, W, _p(x, _fp), cp, _p(out, _fp))
        return out

    def encode(self, kappa):
        kappa = np.ascontiguousarray(kappa, np.float32)
        H, W = kappa.shape
        ctx = [np.zeros((1, self.base, H >> l, W >> l), np.float32) for l in range(self.L)]
        cp = (_fp * self.L)(*[_p(c, _fp) for c in ctx])
        lib().ho_encoder_forward(self.h, H, W, _p(kappa, _fp), cp)
        return ctx


COARSE = {"gmres": 0, "jacobi": 1, "net": 2}


class Hierarchy:
    """Problem hierarchy + V-cycle (inc/multigrid.hpp:70-125)."""

    def __init__(self, kappa2, gamma, omega, lo, hi, levels=3, nu1=1, nu2=1, damping=0.8, alpha=1.0,
                 beta=0.5, coarse="gmres", coarse_iters=10, h=None, coarse_net=None):
        kappa2 = np.ascontiguousarray(kappa2, np.float64)
        gamma = np.ascontiguousarray(gamma, np.float64)
        ny, nx = kappa2.shape
        self.nx, self.ny = nx, ny
        self.h = 1.0 / nx if h is None else h
        self.levels = levels
        self.ptr = lib().ho_mg_create(nx, ny, self.h, omega, _p(kappa2), _p(gamma), lo, hi, levels, nu1, nu2,
                                      damping, alpha, beta, COARSE[coarse], coarse_iters)
        if not self.ptr:
            raise ValueError("bad hierarchy config")
        self._net = coarse_net
        if coarse_net is not None:
            lib().ho_mg_set_coarse_net(self.ptr, coarse_net.h)

    def __del__(self):
        if getattr(self, "ptr", None):
            lib().ho_mg_destroy(self.ptr)
            self.ptr = None

    def level_info(self, l):
        nx, ny, h = C.c_int(), C.c_int(), C.c_double()
        lib().ho_mg_level_info(self.ptr, l, C.byref(nx), C.byref(ny), C.byref(h))
        return nx.value, ny.value, h.value

    def level_coef(self, l):
        nx, ny, _ = self.level_info(l)
        k2 = np.zeros((ny, nx))
        g = np.zeros((ny, nx))
        dA = np.zeros((ny, nx), np.complex128)
        dM = np.zeros((ny, nx), np.complex128)
        lib().ho_mg_level_coef(self.ptr, l, _p(k2), _p(g), cptr(dA), cptr(dM))
        return k2, g, dA, dM

    def apply(self, u, level=0, shifted=False):
        u = cfield(u)
        y = np.zeros_like(u)
        lib().ho_apply(self.ptr, level, int(shifted), cptr(u), cptr(y))
        return y

    def jacobi(self, v, f, damping=0.8, iters=1, level=0, shifted=True):
        v = cfield(v).copy()
        f = cfield(f)
        lib().ho_jacobi(self.ptr, level, int(shifted), cptr(v), cptr(f), damping, iters)
        return v

    def cycle(self, f, v0=None):
        f = cfield(f)
        out = np.zeros_like(f)
        v0p = cptr(cfield(v0)) if v0 is not None else None
        lib().ho_mg_cycle(self.ptr, v0p, cptr(f), cptr(out))
        return out

    def coarse_gmres(self, f, level, iters=10):
        f = cfield(f)
        x = np.zeros_like(f)
        lib().ho_coarse_gmres(self.ptr, level, iters, cptr(f), cptr(x))
        return x


PC = {"v": 0, "vu": 1, "ju": 2}


class Precond:
    def __init__(self, kind, hier, net=None, enc=None):
        self.hier, self.net, self.enc = hier, net, enc
        self.ptr = lib().ho_pc_create(PC[kind], hier.ptr, net.h if net else None, enc.h if enc else None)

    def __del__(self):
        if getattr(self, "ptr", None):
            lib().ho_pc_destroy(self.ptr)
            self.ptr = None

    def apply(self, r):
        r = cfield(r)
        if r.ndim == 2:
            r = r[None]
        z = np.zeros_like(r)
        lib().ho_pc_apply(self.ptr, r.shape[0], cptr(r), cptr(z))
        return z

    def net_guess(self, r):
        r = cfield(r)
        e = np.zeros_like(r)
        lib().ho_pc_net_guess(self.ptr, cptr(r), cptr(e))
        return e

    def ctx(self, l):
        p = lib().ho_pc_ctx(self.ptr, l)
        if not p:
            return None
        nx, ny = self.hier.nx >> l, self.hier.ny >> l
        return np.ctypeslib.as_array(p, shape=(1, self.enc.base, ny, nx)).copy()


def fgmres(pc, B, restart=10, max_iters=200, rel_tol=1e-6, flexible=True, X0=None, nthreads=1):
    """Block FGMRES (inc/krylov.hpp:83-267); returns X, report dict."""
    B = cfield(B)
    nb = B.shape[0]
    X = cfield(X0).copy() if X0 is not None else np.zeros_like(B)
    cap = max_iters + 2
    hist = np.zeros((nb, cap))
    it = np.zeros(nb, np.int32)
    cv = np.zeros(nb, np.int32)
    bk = np.zeros(nb, np.int32)
    hl = np.zeros(nb, np.int32)
    lib().ho_fgmres(pc.ptr, restart, max_iters, rel_tol, int(flexible), nb, cptr(B), cptr(X), _p(hist), cap,
                    _p(it, _ip), _p(cv, _ip), _p(bk, _ip), _p(hl, _ip), nthreads)
    histories = [hist[c, :hl[c]].copy() for c in range(nb)]
    return X, {"iterations": it, "converged": cv.astype(bool), "breakdown": bk.astype(bool),
               "history": histories}


def convergence_factor(hist, target_drop=1e6):
    hist = np.ascontiguousarray(hist, np.float64)
    rho = C.c_double()
    T = lib().ho_convergence_factor(_p(hist), len(hist), target_drop, C.byref(rho))
    return T, rho.value


# ------------------------------------------------ compiled reference (_ref)
_ref = None


def have_ref() -> bool:
    return os.path.exists(REF_PATH)


def ref():
    """The reference headers compiled in place (oracle/build_ref.sh)."""
    global _ref
    if _ref is None:
        if not have_ref():
            raise FileNotFoundError(REF_PATH + " (run oracle/build_ref.sh where /root/reference exists)")
        R = C.CDLL(REF_PATH)
        R.hr_last_error.restype = C.c_char_p
        R.hr_rng_normals.argtypes = [C.c_uint64, C.c_int64, _dp]
        R.hr_rng_u64.argtypes = [C.c_uint64, C.c_int64, C.POINTER(C.c_uint64)]
        R.hr_absorbing_layer.argtypes = [C.c_int, C.c_int, C.c_int, C.c_double, _dp]
        R.hr_restrict.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, _dp, _dp]
        R.hr_synthetic_slowness.argtypes = [C.c_uint64, C.c_int, C.c_int, C.c_double, C.c_double, _dp]
        R.hr_random_rhs_block.argtypes = [C.c_int, C.c_int, C.c_int, C.c_uint64, _dp]
        R.hr_prolong.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, _dp, _dp]
        R.hr_mg_create.restype = _vp
        R.hr_mg_create.argtypes = [C.c_int, C.c_int, C.c_double, _dp, _dp, C.c_double, C.c_double, C.c_int,
                                   C.c_int, C.c_int, C.c_double, C.c_double, C.c_double, C.c_int, C.c_int]
        R.hr_mg_destroy.argtypes = [_vp]
        R.hr_mg_level_coef.argtypes = [_vp, C.c_int, _dp, _dp, _dp, _dp]
        R.hr_apply.argtypes = [_vp, C.c_int, C.c_int, _dp, _dp]
        R.hr_jacobi.argtypes = [_vp, C.c_int, C.c_int, _dp, _dp, C.c_double, C.c_int]
        R.hr_coarse_gmres.argtypes = [_vp, C.c_int, _dp, _dp]
        R.hr_net_create.restype = _vp
        R.hr_net_create.argtypes = [C.c_int] * 5
        R.hr_net_destroy.argtypes = [_vp]
        R.hr_net_nconv.argtypes = [_vp]
        R.hr_net_weight.restype = _fp
        R.hr_net_weight.argtypes = [_vp, C.c_int]
        R.hr_net_bias.restype = _fp
        R.hr_net_bias.argtypes = [_vp, C.c_int]
        R.hr_net_init_he.argtypes = [_vp, C.c_uint64]
        R.hr_net_forward.argtypes = [_vp, C.c_int, C.c_int, C.c_int, _fp, C.POINTER(_fp), _fp]
        R.hr_encoder_forward.argtypes = [_vp, C.c_int, C.c_int, _fp, C.POINTER(_fp)]
        R.hr_conv2d.argtypes = [C.c_int] * 7 + [_fp, _fp, _fp, _fp]
        R.hr_mg_set_coarse_net.argtypes = [_vp, _vp]
        R.hr_pc_create.restype = _vp
        R.hr_pc_create.argtypes = [C.c_int, _vp, _vp, _vp]
        R.hr_pc_destroy.argtypes = [_vp]
        R.hr_pc_apply.argtypes = [_vp, C.c_int, _dp, _dp]
        R.hr_fgmres.argtypes = [_vp, C.c_int, C.c_int, C.c_double, C.c_int, C.c_int, _dp, _dp, _dp, C.c_int,
                                _ip, _ip, _ip, _ip, C.c_int, _dp]
        R.hr_paper_create.restype = _vp
        R.hr_paper_create.argtypes = [C.c_int] * 7 + [C.c_uint64]
        R.hr_paper_destroy.argtypes = [_vp]
        R.hr_paper_zero_shifts.argtypes = [_vp]
        R.hr_paper_save.argtypes = [_vp, C.c_char_p, C.c_char_p]
        R.hr_paper_load.argtypes = [_vp, C.c_char_p]
        R.hr_paper_encode.argtypes = [_vp, C.c_int, C.c_int, _dp]
        R.hr_paper_forward.argtypes = [_vp, C.c_int, C.c_int, C.c_int, _fp, _fp]
        R.hr_paper_feature.argtypes = [_vp, C.c_int, _fp]
        R.hr_paper_pc_create.restype = _vp
        R.hr_paper_pc_create.argtypes = [C.c_int, _vp, _vp]
        R.hr_paper_pc_destroy.argtypes = [_vp]
        R.hr_paper_pc_apply.argtypes = [_vp, C.c_int, _dp, _dp]
        R.hr_paper_fgmres.argtypes = [_vp, C.c_int, C.c_int, C.c_double, C.c_int, _dp, _dp, _dp, C.c_int, _ip, _ip]
        R.hr_gen_sample_pair.argtypes = [_vp, C.c_uint64, C.c_int, C.c_int, _dp, _dp]
        R.hr_paper_trainable_count.argtypes = [_vp]
        R.hr_paper_trainable_count.restype = C.c_int64
        R.hr_paper_train_batch.argtypes = [_vp, C.c_int, C.c_int, C.c_int, _fp, _fp, _fp, C.c_int, C.c_int, C.c_int,
                                           C.c_double, _dp, _fp, _fp]
        R.hr_paper_train.argtypes = [_vp, C.c_int, C.c_double, C.c_int, C.c_int, C.c_double, C.c_int, C.c_uint64,
                                     C.c_int, C.c_int, C.c_int, _fp, _fp, _ip, C.c_int, _dp, _dp, _dp, C.c_int, _ip,
                                     _ip]
        R.hr_paper_retrain.argtypes = [_vp, _vp, C.c_int, C.c_int, C.c_double, C.c_int, C.c_uint64, _dp, C.c_int, _ip,
                                       _ip]
        R.hr_write_slw1.argtypes = [C.c_char_p, C.c_int, C.c_int, _dp]
        R.hr_read_slw1.argtypes = [C.c_char_p, _ip, _ip, _dp]
        R.hr_init()
        _ref = R
    return _ref


def ref_synthetic_slowness(seed, nx, ny, lo=0.25, hi=1.0):
    """inc/datagen.hpp:94-119 (the reference build)."""
    out = np.zeros((ny, nx))
    _rcheck(ref().hr_synthetic_slowness(seed, nx, ny, lo, hi, _p(out)))
    return out


def ref_random_rhs_block(nx, ny, count, seed):
    """inc/bench.hpp:83-90 (the reference build)."""
    out = np.zeros((count, ny, nx), np.complex128)
    _rcheck(ref().hr_random_rhs_block(nx, ny, count, seed, cptr(out)))
    return out


def _rcheck(rc):
    if rc != 0:
        raise RuntimeError(ref().hr_last_error().decode())


class RefNet:
    def __init__(self, kind, L, base, in_ch, ctx_ch=0, seed=None):
        self.kind, self.L, self.base, self.in_ch, self.ctx_ch = kind, L, base, in_ch, ctx_ch
        self.h = ref().hr_net_create(kind, L, base, in_ch, ctx_ch)
        if seed is not None:
            ref().hr_net_init_he(self.h, seed)

    def __del__(self):
        if getattr(self, "h", None):
            ref().hr_net_destroy(self.h)
            self.h = None

    def convs(self):
        out = []
        nets = UNet(self.kind, self.L, self.base, self.in_ch, self.ctx_ch)  # shapes only
        for i, (w, b) in enumerate(nets.convs()):
            wv = np.ctypeslib.as_array(ref().hr_net_weight(self.h, i), shape=w.shape)
            bv = np.ctypeslib.as_array(ref().hr_net_bias(self.h, i), shape=b.shape)
            out.append((wv, bv))
        return out

    def forward(self, x, ctx=None):
        x = np.ascontiguousarray(x, np.float32)
        B, _, H, W = x.shape
        out = np.zeros((B, 2, H, W), np.float32)
        cp = None
        if ctx is not None:
            ctx = [np.ascontiguousarray(c, np.float32) for c in ctx]
            cp = (_fp * len(ctx))(*[_p(c, _fp) for c in ctx])
        _rcheck(ref().hr_net_forward(self.h, B, H, W, _p(x, _fp), cp, _p(out, _fp)))
        return out

    def encode(self, kappa):
        kappa = np.ascontiguousarray(kappa, np.float32)
        H, W = kappa.shape
        ctx = [np.zeros((1, self.base, H >> l, W >> l), np.float32) for l in range(self.L)]
        cp = (_fp * self.L)(*[_p(c, _fp) for c in ctx])
        _rcheck(ref().hr_encoder_forward(self.h, H, W, _p(kappa, _fp), cp))
        return ctx


class RefHierarchy:
    def __init__(self, kappa2, gamma, omega, lo, hi, levels=3, nu1=1, nu2=1, damping=0.8, alpha=1.0, beta=0.5,
                 coarse="gmres", coarse_iters=10, coarse_net=None):
        kappa2 = np.ascontiguousarray(kappa2, np.float64)
        gamma = np.ascontiguousarray(gamma, np.float64)
        self.ny, self.nx = kappa2.shape
        kind = {"gmres": 0, "jacobi": 1, "net": 2, "dense": 3}[coarse]
        self.ptr = ref().hr_mg_create(self.nx, self.ny, omega, _p(kappa2), _p(gamma), lo, hi, levels, nu1, nu2,
                                      damping, alpha, beta, kind, coarse_iters)
        if not self.ptr:
            raise ValueError(ref().hr_last_error().decode())
        self._net = coarse_net
        if coarse_net is not None:
            ref().hr_mg_set_coarse_net(self.ptr, coarse_net.h)

    def __del__(self):
        if getattr(self, "ptr", None):
            ref().hr_mg_destroy(self.ptr)
            self.ptr = None

    def level_coef(self, l):
        nx, ny = self.nx >> l, self.ny >> l
        k2 = np.zeros((ny, nx))
        g = np.zeros((ny, nx))
        dA = np.zeros((ny, nx), np.complex128)
        dM = np.zeros((ny, nx), np.complex128)
        ref().hr_mg_level_coef(self.ptr, l, _p(k2), _p(g), cptr(dA), cptr(dM))
        return k2, g, dA, dM

    def apply(self, u, level=0, shifted=False):
        u = cfield(u)
        y = np.zeros_like(u)
        _rcheck(ref().hr_apply(self.ptr, level, int(shifted), cptr(u), cptr(y)))
        return y

    def jacobi(self, v, f, damping=0.8, iters=1, level=0, shifted=True):
        v = cfield(v).copy()
        _rcheck(ref().hr_jacobi(self.ptr, level, int(shifted), cptr(v), cptr(cfield(f)), damping, iters))
        return v

    def coarse_gmres(self, f, level):
        f = cfield(f)
        x = np.zeros_like(f)
        _rcheck(ref().hr_coarse_gmres(self.ptr, level, cptr(f), cptr(x)))
        return x


class RefPrecond:
    def __init__(self, kind, hier, net=None, enc=None):
        self.hier, self.net, self.enc = hier, net, enc
        self.ptr = ref().hr_pc_create(PC[kind], hier.ptr, net.h if net else None, enc.h if enc else None)

    def __del__(self):
        if getattr(self, "ptr", None):
            ref().hr_pc_destroy(self.ptr)
            self.ptr = None

    def apply(self, r):
        r = cfield(r)
        if r.ndim == 2:
            r = r[None]
        z = np.zeros_like(r)
        _rcheck(ref().hr_pc_apply(self.ptr, r.shape[0], cptr(r), cptr(z)))
        return z


def ref_fgmres(pc, B, restart=10, max_iters=200, rel_tol=1e-6, flexible=True, nthreads=1):
    B = cfield(B)
    nb = B.shape[0]
    X = np.zeros_like(B)
    cap = max_iters + 2
    hist = np.zeros((nb, cap))
    it = np.zeros(nb, np.int32)
    cv = np.zeros(nb, np.int32)
    bk = np.zeros(nb, np.int32)
    hl = np.zeros(nb, np.int32)
    secs = C.c_double()
    _rcheck(ref().hr_fgmres(pc.ptr, restart, max_iters, rel_tol, int(flexible), nb, cptr(B), cptr(X), _p(hist), cap,
                            _p(it, _ip), _p(cv, _ip), _p(bk, _ip), _p(hl, _ip), nthreads, C.byref(secs)))
    histories = [hist[c, :hl[c]].copy() for c in range(nb)]
    return X, {"iterations": it, "converged": cv.astype(bool), "breakdown": bk.astype(bool), "history": histories,
               "seconds": secs.value}


def ref_conv2d(x, w, b, stride=1):
    x = np.ascontiguousarray(x, np.float32)
    w = np.ascontiguousarray(w, np.float32)
    b = np.ascontiguousarray(b, np.float32)
    N, cin, H, W = x.shape
    cout, _, k, _ = w.shape
    Ho = (H + 2 * ((k - 1) // 2) - k) // stride + 1
    Wo = (W + 2 * ((k - 1) // 2) - k) // stride + 1
    y = np.zeros((N, cout, Ho, Wo), np.float32)
    _rcheck(ref().hr_conv2d(N, cin, cout, H, W, k, stride, _p(x, _fp), _p(w, _fp), _p(b, _fp), _p(y, _fp)))
    return y


class RefPaperNet:
    """The reference's paper U-Net (inc/unet.hpp:113-295) with seeded weights
    and seeded batch-norm buffers (ref_capi.cpp hr_paper_create)."""

    def __init__(self, levels=3, base=8, rpl=1, bot=1, kud=5, kres=3, variant=0, seed=77):
        self.variant = variant
        self.h = ref().hr_paper_create(levels, base, rpl, bot, kud, kres, variant, seed)
        if not self.h:
            raise ValueError(ref().hr_last_error().decode())

    def __del__(self):
        if getattr(self, "h", None):
            ref().hr_paper_destroy(self.h)
            self.h = None

    def zero_shifts(self):
        ref().hr_paper_zero_shifts(self.h)

    def save(self, path, digest="helmbench"):
        _rcheck(ref().hr_paper_save(self.h, path.encode(), digest.encode()))

    def encode(self, kappa2):
        k = np.ascontiguousarray(kappa2, np.float64)
        _rcheck(ref().hr_paper_encode(self.h, k.shape[1], k.shape[0], _p(k)))

    def forward(self, x):
        x = np.ascontiguousarray(x, np.float32)
        B, _, H, W = x.shape
        y = np.zeros((B, 2, H, W), np.float32)
        _rcheck(ref().hr_paper_forward(self.h, B, H, W, _p(x, _fp), _p(y, _fp)))
        return y


def _paper_train_methods():
    def train_batch(self, x, target, kappa=None, train_mode=True, with_grad=True, step=False, lr=1e-4):
        """traindet::run_batch (+ adam_step) -> (loss, out, trainable grads concatenated)"""
        x = np.ascontiguousarray(x, np.float32)
        t = np.ascontiguousarray(target, np.float32)
        k = None if kappa is None else np.ascontiguousarray(kappa, np.float32)
        B, _, H, W = x.shape
        out = np.zeros((B, 2, H, W), np.float32)
        g = np.zeros(ref().hr_paper_trainable_count(self.h), np.float32)
        loss = C.c_double()
        _rcheck(ref().hr_paper_train_batch(self.h, B, H, W, _p(x, _fp), _p(k, _fp) if k is not None else None,
                                           _p(t, _fp), int(train_mode), int(with_grad), int(step), lr, C.byref(loss),
                                           _p(out, _fp), _p(g, _fp)))
        return loss.value, out, g

    def train(self, epochs, lr0, batch0, t0, val_fraction, es, seed, r_hat, e_true, model_id, kappa2, gamma):
        r = np.ascontiguousarray(r_hat, np.float32)
        e = np.ascontiguousarray(e_true, np.float32)
        m = np.ascontiguousarray(model_id, np.int32)
        k2 = np.ascontiguousarray(kappa2, np.float64)
        gm = np.ascontiguousarray(gamma, np.float64)
        N, _, H, W = r.shape
        h = np.zeros((max(epochs, 1), 4))
        n, ab = C.c_int(), C.c_int()
        _rcheck(ref().hr_paper_train(self.h, epochs, lr0, batch0, t0, val_fraction, int(es), seed, N, H, W, _p(r, _fp),
                                     _p(e, _fp), _p(m, _ip), k2.shape[0], _p(k2), _p(gm), _p(h), h.shape[0],
                                     C.byref(n), C.byref(ab)))
        return h[:n.value], bool(ab.value)

    def retrain(self, hier, n_pairs, epochs, lr0, es, seed):
        h = np.zeros((max(epochs, 1), 4))
        n, ab = C.c_int(), C.c_int()
        _rcheck(ref().hr_paper_retrain(self.h, hier.ptr, n_pairs, epochs, lr0, int(es), seed, _p(h), h.shape[0],
                                       C.byref(n), C.byref(ab)))
        return h[:n.value], bool(ab.value)

    RefPaperNet.train_batch = train_batch
    RefPaperNet.train = train
    RefPaperNet.retrain = retrain


_paper_train_methods()


class RefPaperPrecond:
    """kind "ju": JacobiUnetPreconditioner, "vu": UnetVCyclePreconditioner (inc/precond.hpp:104-165)."""

    def __init__(self, kind, hier, net):
        self.hier, self.net = hier, net
        self.nx, self.ny = hier.nx, hier.ny
        self.h = ref().hr_paper_pc_create({"ju": 0, "vu": 1}[kind], hier.ptr, net.h)
        if not self.h:
            raise ValueError(ref().hr_last_error().decode())

    def __del__(self):
        if getattr(self, "h", None):
            ref().hr_paper_pc_destroy(self.h)
            self.h = None

    def apply(self, r):
        r = np.ascontiguousarray(r, np.complex128)
        z = np.zeros_like(r)
        _rcheck(ref().hr_paper_pc_apply(self.h, r.shape[0], cptr(r), cptr(z)))
        return z

    def fgmres(self, B, restart=10, max_iters=20, rel_tol=1e-6):
        B = np.ascontiguousarray(B, np.complex128)
        nb = B.shape[0]
        X = np.zeros_like(B)
        cap = max_iters + 2
        hist = np.zeros((nb, cap))
        it = np.zeros(nb, np.int32)
        hl = np.zeros(nb, np.int32)
        _rcheck(ref().hr_paper_fgmres(self.h, restart, max_iters, rel_tol, nb, cptr(B), cptr(X), _p(hist), cap,
                                      _p(it, _ip), _p(hl, _ip)))
        return X, [hist[c, :hl[c]].copy() for c in range(nb)], it


def ref_gen_sample_pair(hier, seed, k_forced=-1, k_max=10):
    """gen_sample_pair (inc/datagen.hpp:191-219) of the reference: (r, e)."""
    r = np.zeros((hier.ny, hier.nx), np.complex128)
    e = np.zeros_like(r)
    _rcheck(ref().hr_gen_sample_pair(hier.ptr, seed, k_forced, k_max, cptr(r), cptr(e)))
    return r, e


def block_fgmres_np(apply_A, apply_M, B, restart=10, max_iters=200, rel_tol=1e-6):
    """Block flexible GMRES (one block Krylov space for all columns of B) in
    fp64 numpy -- the oracle for hb_block_fgmres.  A restatement of the
    published algorithm (Saad, Iterative Methods 2nd ed. 6.12 / 9.4.1, with a
    flexible Z): restart from R = B - A X = V_0 S (QR), per step Z_j = M V_j,
    W = A Z_j, block CGS2 against V_0..V_j, W = V_{j+1} H_{j+1,j} (QR), the
    per-column residual of the block least-squares problem
    min_Y ||[S; 0] - Hbar Y||.  apply_A / apply_M map (p, ny, nx) -> (p, ny, nx).
    Returns X, per-column histories ([0] = ||b_c||), block steps."""
    B = np.asarray(B, np.complex128)
    p = B.shape[0]
    shp = B.shape
    N = B[0].size
    m = restart
    X = np.zeros((N, p), np.complex128)
    beta0 = np.linalg.norm(B.reshape(p, N), axis=1)
    hist = [[float(b)] for b in beta0]
    it = 0
    while True:
        R = (B - apply_A(X.T.reshape(shp))).reshape(p, N).T
        Q, S = np.linalg.qr(R)
        V = [Q]
        Z = []
        H = np.zeros(((m + 1) * p, m * p), np.complex128)
        E = np.zeros(((m + 1) * p, p), np.complex128)
        E[:p] = S
        done = False
        k = 0
        for j in range(m):
            Zj = apply_M(V[j].T.reshape(shp)).reshape(p, N).T
            W = apply_A(Zj.T.reshape(shp)).reshape(p, N).T
            Va = np.concatenate(V, axis=1)
            for _ in range(2):
                Hc = Va.conj().T @ W
                W = W - Va @ Hc
                H[:(j + 1) * p, j * p:(j + 1) * p] += Hc
            Qn, Rn = np.linalg.qr(W)
            H[(j + 1) * p:(j + 2) * p, j * p:(j + 1) * p] = Rn
            V.append(Qn)
            Z.append(Zj)
            it += 1
            k = j + 1
            Hs, Es = H[:(k + 1) * p, :k * p], E[:(k + 1) * p]
            Y = np.linalg.lstsq(Hs, Es, rcond=None)[0]
            res = np.linalg.norm(Es - Hs @ Y, axis=0)
            for c in range(p):
                hist[c].append(float(res[c]))
            if np.all(res <= rel_tol * beta0) or it >= max_iters:
                done = True
                break
        Hs, Es = H[:(k + 1) * p, :k * p], E[:(k + 1) * p]
        Y = np.linalg.lstsq(Hs, Es, rcond=None)[0]
        X = X + np.concatenate(Z, axis=1) @ Y
        if done:
            return X.T.reshape(shp), [np.array(h) for h in hist], it
