"""Python host mirror of the helmbench solver/preconditioner API over the
libhelmgpu C ABI (include/helmgpu.h).

Names follow the reference (inc/ = /root/reference/proj/include/helmbench/):
KrylovConfig / SolveReport (inc/krylov.hpp:11-35), VCycleConfig
(inc/multigrid.hpp:13-21), Preconditioner and its plugins
(inc/precond.hpp:14-165), block_fgmres (inc/krylov.hpp:83).  Errors keep the
reference's convention: contract violations raise ValueError (the C++
std::invalid_argument), numerical/device failures raise RuntimeError.

There is no CPU fallback: importing this module on a machine without the
built library raises, and every compute call goes through the CUDA library.
"""
from __future__ import annotations

import ctypes as C
import dataclasses
import os
from typing import List, Optional, Sequence

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libhelmgpu.so")

_dp = C.POINTER(C.c_double)
_fp = C.POINTER(C.c_float)
_ip = C.POINTER(C.c_int)
_u8p = C.POINTER(C.c_uint8)
_vp = C.c_void_p

HB_COARSE = {"gmres": 0, "jacobi": 1, "net": 2, "dense": 3}
HB_PC = {"v": 0, "vu": 1, "ju": 2}


class _VCycleCfg(C.Structure):
    _fields_ = [("levels", C.c_int), ("nu1", C.c_int), ("nu2", C.c_int), ("damping", C.c_double),
                ("alpha", C.c_double), ("beta", C.c_double), ("coarse_solver", C.c_int),
                ("coarse_iters", C.c_int)]


class _NetCfg(C.Structure):
    _fields_ = [("kind", C.c_int), ("levels", C.c_int), ("base", C.c_int), ("in_ch", C.c_int),
                ("ctx_ch", C.c_int)]


class _UNetCfg(C.Structure):
    _fields_ = [("levels", C.c_int), ("base_channels", C.c_int), ("resnet_per_level", C.c_int),
                ("bottleneck_resnets", C.c_int), ("updown_kernel", C.c_int), ("res_kernel", C.c_int)]


class _TrainCfg(C.Structure):  # hb_train_cfg (TrainConfig, inc/training.hpp:12-20)
    _fields_ = [("epochs", C.c_int), ("lr0", C.c_double), ("batch0", C.c_int), ("t0", C.c_int),
                ("val_fraction", C.c_double), ("encoder_solver", C.c_int), ("seed", C.c_uint64)]


class _KrylovCfg(C.Structure):
    _fields_ = [("restart", C.c_int), ("max_iters", C.c_int), ("rel_tol", C.c_double), ("flexible", C.c_int)]


_lib = None


def lib():
    """Load libhelmgpu.so (fails loudly when it has not been built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} missing: run `python -m paper_2203_11025_b200.build` "
                              "(the CUDA library is the only implementation; there is no CPU fallback)")
        # HB_LIB_PATH: load another build of the same library (A/B timing, tools/abbuild.sh)
        L = C.CDLL(os.environ.get("HB_LIB_PATH", LIB_PATH))
        L.hb_create.argtypes = [C.c_int, C.POINTER(_vp)]
        L.hb_destroy.argtypes = [_vp]
        L.hb_last_error.restype = C.c_char_p
        L.hb_last_error.argtypes = [_vp]
        L.hb_stream.restype = _vp
        L.hb_stream.argtypes = [_vp]
        L.hb_synchronize.argtypes = [_vp]
        L.hb_set_problem.argtypes = [_vp, C.c_int, C.c_int, C.c_double, C.c_double, _dp, _dp, C.c_double, C.c_double]
        L.hb_build_hierarchy.argtypes = [_vp, C.POINTER(_VCycleCfg)]
        L.hb_level_info.argtypes = [_vp, C.c_int, _ip, _ip, _dp]
        L.hb_set_net.argtypes = [_vp, C.c_int, C.POINTER(_NetCfg)]
        L.hb_net_num_convs.argtypes = [_vp, C.c_int]
        L.hb_net_conv_shape.argtypes = [_vp, C.c_int, C.c_int, _ip, _ip]
        L.hb_load_conv.argtypes = [_vp, C.c_int, C.c_int, _fp, _fp]
        L.hb_get_conv.argtypes = [_vp, C.c_int, C.c_int, _fp, _fp]
        L.hb_init_net_he.argtypes = [_vp, C.c_int, C.c_uint64]
        L.hb_net_forward.argtypes = [_vp, C.c_int, C.c_int, C.c_int, _fp, _fp]
        L.hb_encode.argtypes = [_vp]
        L.hb_get_context.argtypes = [_vp, C.c_int, _fp]
        L.hb_operator_apply.argtypes = [_vp, C.c_int, C.c_int, C.c_int, _dp, _dp]
        L.hb_jacobi.argtypes = [_vp, C.c_int, C.c_int, _dp, _dp, C.c_int]
        L.hb_restrict.argtypes = [_vp, C.c_int, C.c_int, _dp, _dp]
        L.hb_prolong.argtypes = [_vp, C.c_int, C.c_int, _dp, _dp]
        L.hb_coarse_solve.argtypes = [_vp, C.c_int, _dp, _dp]
        L.hb_precond_apply.argtypes = [_vp, C.c_int, C.c_int, _dp, _dp]
        L.hb_precond_apply_device.argtypes = [_vp, C.c_int, C.c_int, _vp, _vp]
        L.hb_precond_name.restype = C.c_char_p
        L.hb_precond_name.argtypes = [C.c_int]
        L.hb_precond_requires_flexible.argtypes = [_vp, C.c_int]
        L.hb_fgmres.argtypes = [_vp, C.POINTER(_KrylovCfg), C.c_int, C.c_int, _dp, _dp, _dp, _dp, C.c_int, _ip, _ip,
                                _u8p, _u8p]
        L.hb_block_fgmres.argtypes = [_vp, C.POINTER(_KrylovCfg), C.c_int, C.c_int, _dp, _dp, _dp, _dp, C.c_int, _ip, _ip,
                                _u8p, _u8p]
        L.hb_fgmres_device.argtypes = [_vp, C.POINTER(_KrylovCfg), C.c_int, C.c_int, _vp, _vp, _dp, C.c_int, _ip,
                                       _ip, _u8p, _u8p]
        L.hb_set_paper_net.argtypes = [_vp, C.POINTER(_UNetCfg), C.c_int]
        L.hb_paper_init.argtypes = [_vp, C.c_uint64]
        L.hb_paper_param_count.argtypes = [_vp]
        L.hb_paper_param_info.argtypes = [_vp, C.c_int, C.c_char_p, C.c_int, _ip]
        L.hb_paper_param.argtypes = [_vp, C.c_char_p, C.c_int64, _fp, _fp]
        L.hb_load_checkpoint.argtypes = [_vp, C.c_char_p]
        L.hb_save_checkpoint.argtypes = [_vp, C.c_char_p, C.c_char_p]
        L.hb_paper_forward.argtypes = [_vp, C.c_int, C.c_int, C.c_int, _fp, _fp]
        L.hb_gen_sample_pairs.argtypes = [_vp, C.c_int, C.POINTER(C.c_uint64), C.c_int, C.c_int, _dp, _dp, _ip]
        L.hb_paper_train_batch.argtypes = [_vp, C.c_int, C.c_int, C.c_int, _fp, _fp, _fp, C.c_int, C.c_int, C.c_int,
                                           C.c_double, _dp, _fp]
        L.hb_paper_trainable_count.argtypes = [_vp]
        L.hb_paper_trainable_count.restype = C.c_int64
        L.hb_paper_grads.argtypes = [_vp, C.c_int64, _fp]
        L.hb_paper_set_trainable_prefix.argtypes = [_vp, C.c_char_p, C.c_int]
        L.hb_paper_adam_reset.argtypes = [_vp]
        L.hb_paper_train.argtypes = [_vp, C.POINTER(_TrainCfg), C.c_int, C.c_int, C.c_int, _fp, _fp, _ip, C.c_int,
                                     _dp, _dp, _dp, C.c_int, _ip, _ip]
        L.hb_paper_retrain.argtypes = [_vp, C.c_int, C.c_int, C.POINTER(_TrainCfg), C.c_uint64, _dp, C.c_int, _ip,
                                       _ip]
        L.hb_write_slw1.argtypes = [C.c_char_p, C.c_int, C.c_int, _dp]
        L.hb_read_slw1.argtypes = [C.c_char_p, _ip, _ip, _dp]
        L.hb_slab_partition.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, _ip, _ip]
        L.hb_nccl_unique_id.argtypes = [C.c_char_p]
        L.hb_slab_init_nccl.argtypes = [_vp, C.c_int, C.c_int, C.c_char_p]
        L.hb_slab_init_local.argtypes = [C.POINTER(_vp), C.c_int]
        L.hb_slab_rows.argtypes = [_vp, _ip, _ip]
        L.hb_precond_apply_slab.argtypes = [_vp, C.c_int, C.c_int, _dp, _dp]
        L.hb_fgmres_slab.argtypes = [_vp, C.POINTER(_KrylovCfg), C.c_int, C.c_int, _dp, _dp, _dp, _dp, C.c_int, _ip,
                                     _ip, _u8p, _u8p]
        L.hb_rng_normals.argtypes = [C.c_uint64, C.c_int64, _dp]
        L.hb_absorbing_layer.argtypes = [C.c_int, C.c_int, C.c_int, C.c_double, _dp]
        L.hb_make_medium.argtypes = [C.c_int, C.c_int, C.c_uint64, C.c_double, C.c_double, C.c_double, C.c_int,
                                     C.c_uint64, C.c_int, C.c_double, C.c_double, _dp]
        L.hb_point_sources.argtypes = [C.c_uint64, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, _ip, _ip]
        L.hb_set_option.argtypes = [_vp, C.c_char_p, C.c_int64]
        L.hb_prof_enable.argtypes = [_vp, C.c_int]
        L.hb_prof_reset.argtypes = [_vp]
        L.hb_prof_count.argtypes = [_vp]
        L.hb_prof_name.restype = C.c_char_p
        L.hb_prof_name.argtypes = [_vp, C.c_int]
        L.hb_prof_get.argtypes = [_vp, C.c_int, _dp, C.POINTER(C.c_int64), _dp, _dp]
        L.hb_prof_detail.argtypes = [_vp, C.c_int, C.c_char_p, C.c_int]
        L.hb_launch_count.restype = C.c_int64
        L.hb_launch_count.argtypes = [_vp]
        _lib = L
    return _lib


def _p(a, t=_dp):
    return None if a is None else a.ctypes.data_as(t)


def _c128(a):
    return np.ascontiguousarray(a, dtype=np.complex128)


# ------------------------------------------------------------ config types
@dataclasses.dataclass
class KrylovConfig:  # inc/krylov.hpp:11-16
    restart: int = 10
    max_iters: int = 200
    rel_tol: float = 1e-6
    flexible: bool = True


@dataclasses.dataclass
class VCycleConfig:  # inc/multigrid.hpp:13-21
    levels: int = 3
    nu1: int = 1
    nu2: int = 1
    damping: float = 0.8
    alpha: float = 1.0
    beta: float = 0.5
    coarse_iters: int = 10
    coarse_solver: str = "gmres"  # gmres | jacobi | net


@dataclasses.dataclass
class UNetConfig:  # inc/unet.hpp:113-120 (the paper's network)
    levels: int = 3
    base_channels: int = 16
    resnet_per_level: int = 1
    bottleneck_resnets: int = 3
    updown_kernel: int = 5
    res_kernel: int = 3


NET_VARIANT = {"standalone": 0, "encoder_solver": 1}  # NetVariant, inc/precond.hpp:55


@dataclasses.dataclass
class TrainConfig:  # inc/training.hpp:12-20
    epochs: int = 40
    lr0: float = 1e-4
    batch0: int = 20
    t0: int = 48
    val_fraction: float = 0.1
    encoder_solver: bool = False
    seed: int = 1

    def _c(self):
        return _TrainCfg(self.epochs, self.lr0, self.batch0, self.t0, self.val_fraction, int(self.encoder_solver),
                         self.seed)


@dataclasses.dataclass
class TrainHistory:  # inc/training.hpp:48-59
    epochs: list  # [(epoch, mean_rel_error_train, mean_rel_error_val, lr, batch)]
    aborted_non_finite: bool = False

    def write_csv(self, f):
        f.write("epoch,mean_rel_error_train,mean_rel_error_val,lr,batch\n")
        for e in self.epochs:
            f.write(f"{e[0]},{_g6(e[1])},{_g6(e[2])},{_g6(e[3])},{e[4]}\n")


def _g6(x):  # std::ostream default (6 significant digits)
    return f"{x:.6g}"


@dataclasses.dataclass
class SolveReport:  # inc/krylov.hpp:20-35
    residual_history: List[np.ndarray]
    iterations: List[int]
    converged: List[bool]
    breakdown: List[bool]

    def write_csv(self, os_):
        os_.write("iter,rhs_index,relative_residual\n")
        for c, h in enumerate(self.residual_history):
            r0 = h[0] if len(h) and h[0] > 0 else 1.0
            for i, v in enumerate(h):
                os_.write(f"{i},{c},{v / r0:g}\n")  # operator<< default: 6 significant digits


# ------------------------------------------------------------------ context
class Context:
    """One GPU context (hb_ctx): problem, hierarchy, nets, solver state."""

    def __init__(self, device: int = 0):
        h = _vp()
        rc = lib().hb_create(device, C.byref(h))
        if rc != 0:
            raise RuntimeError("hb_create: " + lib().hb_last_error(None).decode())
        self.h = h
        self.nx = self.ny = 0
        self.vcfg: Optional[VCycleConfig] = None

    def close(self):
        if getattr(self, "h", None):
            lib().hb_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except TypeError:  # interpreter shutdown: module globals already cleared
            pass

    def _check(self, rc):
        if rc != 0:
            msg = lib().hb_last_error(self.h).decode()
            if rc == -1:
                raise ValueError(msg)
            raise RuntimeError(msg)

    @property
    def stream(self) -> int:
        return lib().hb_stream(self.h) or 0

    def synchronize(self):
        self._check(lib().hb_synchronize(self.h))

    # problem + hierarchy (inc/grid.hpp:128, inc/multigrid.hpp:72)
    def set_problem(self, kappa2, gamma, omega, lo, hi, h=None):
        kappa2 = np.ascontiguousarray(kappa2, np.float64)
        gamma = np.ascontiguousarray(gamma, np.float64)
        ny, nx = kappa2.shape
        self.nx, self.ny = nx, ny
        self.h_mesh = 1.0 / nx if h is None else h
        self._check(lib().hb_set_problem(self.h, nx, ny, self.h_mesh, omega, _p(kappa2), _p(gamma), lo, hi))

    def build_hierarchy(self, cfg: VCycleConfig):
        c = _VCycleCfg(cfg.levels, cfg.nu1, cfg.nu2, cfg.damping, cfg.alpha, cfg.beta,
                       HB_COARSE[cfg.coarse_solver], cfg.coarse_iters)
        self._check(lib().hb_build_hierarchy(self.h, C.byref(c)))
        self.vcfg = cfg

    def level_info(self, l):
        nx, ny, h = C.c_int(), C.c_int(), C.c_double()
        self._check(lib().hb_level_info(self.h, l, C.byref(nx), C.byref(ny), C.byref(h)))
        return nx.value, ny.value, h.value

    # networks
    def set_net(self, slot, kind, levels, base=16, in_ch=3, ctx_ch=0):
        c = _NetCfg({"solver": 0, "encoder": 1}[kind], levels, base, in_ch, ctx_ch)
        self._check(lib().hb_set_net(self.h, slot, C.byref(c)))

    def init_net_he(self, slot, seed):
        self._check(lib().hb_init_net_he(self.h, slot, seed))

    def net_convs(self, slot):
        out = []
        for i in range(lib().hb_net_num_convs(self.h, slot)):
            co, ci = C.c_int(), C.c_int()
            self._check(lib().hb_net_conv_shape(self.h, slot, i, C.byref(co), C.byref(ci)))
            w = np.zeros((co.value, ci.value, 3, 3), np.float32)
            b = np.zeros(co.value, np.float32)
            self._check(lib().hb_get_conv(self.h, slot, i, _p(w, _fp), _p(b, _fp)))
            out.append((w, b))
        return out

    def load_net(self, slot, convs):
        for i, (w, b) in enumerate(convs):
            w = np.ascontiguousarray(w, np.float32)
            b = np.ascontiguousarray(b, np.float32)
            self._check(lib().hb_load_conv(self.h, slot, i, _p(w, _fp), _p(b, _fp)))

    def net_forward(self, x):
        x = np.ascontiguousarray(x, np.float32)
        B, _, H, W = x.shape
        y = np.zeros((B, 2, H, W), np.float32)
        self._check(lib().hb_net_forward(self.h, B, H, W, _p(x, _fp), _p(y, _fp)))
        return y

    # the paper's U-Net (inc/unet.hpp:113-295) -- the network of M_JU / M_VU once set
    def set_paper_net(self, cfg: UNetConfig, variant: str = "standalone"):
        c = _UNetCfg(cfg.levels, cfg.base_channels, cfg.resnet_per_level, cfg.bottleneck_resnets,
                     cfg.updown_kernel, cfg.res_kernel)
        self._check(lib().hb_set_paper_net(self.h, C.byref(c), NET_VARIANT[variant]))

    def paper_init(self, seed: int):
        self._check(lib().hb_paper_init(self.h, seed))

    def paper_params(self):
        """[(name, (n, c, h, w))] in the reference's registry order."""
        out = []
        buf = C.create_string_buffer(256)
        d = (C.c_int * 4)()
        for i in range(lib().hb_paper_param_count(self.h)):
            self._check(lib().hb_paper_param_info(self.h, i, buf, 256, d))
            out.append((buf.value.decode(), tuple(d)))
        return out

    def paper_param(self, name: str, value=None):
        dims = dict(self.paper_params())[name]
        out = np.zeros(dims, np.float32)
        inp = None if value is None else np.ascontiguousarray(value, np.float32).reshape(dims)
        self._check(lib().hb_paper_param(self.h, name.encode(), out.size, _p(inp, _fp) if inp is not None else None,
                                         _p(out, _fp)))
        return out

    def load_checkpoint(self, path: str):  # inc/checkpoint.hpp:83-104
        self._check(lib().hb_load_checkpoint(self.h, os.fspath(path).encode()))

    def save_checkpoint(self, path: str, digest: str = ""):  # inc/checkpoint.hpp:57-78
        self._check(lib().hb_save_checkpoint(self.h, os.fspath(path).encode(), digest.encode()))

    def paper_forward(self, x):
        x = np.ascontiguousarray(x, np.float32)
        B, _, H, W = x.shape
        y = np.zeros((B, 2, H, W), np.float32)
        self._check(lib().hb_paper_forward(self.h, B, H, W, _p(x, _fp), _p(y, _fp)))
        return y

    # training (inc/training.hpp:121-298, inc/adam.hpp:25-58) on the device
    def paper_train_batch(self, x, target, kappa=None, train_mode=True, with_grad=True, step=False, lr=1e-4):
        """run_batch (+ adam_step): x [B][4][H][W], target [B][2][H][W] -> (loss, out)"""
        x = np.ascontiguousarray(x, np.float32)
        t = np.ascontiguousarray(target, np.float32)
        k = None if kappa is None else np.ascontiguousarray(kappa, np.float32)
        B, _, H, W = x.shape
        out = np.zeros((B, 2, H, W), np.float32)
        loss = C.c_double()
        self._check(lib().hb_paper_train_batch(self.h, B, H, W, _p(x, _fp), _p(k, _fp) if k is not None else None,
                                               _p(t, _fp), int(train_mode), int(with_grad), int(step), lr,
                                               C.byref(loss), _p(out, _fp)))
        return loss.value, out

    def paper_grads(self):
        """the last batch's trainable gradients {name: array} (registry order)"""
        n = lib().hb_paper_trainable_count(self.h)
        g = np.zeros(n, np.float32)
        self._check(lib().hb_paper_grads(self.h, n, _p(g, _fp)))
        return g

    def paper_set_trainable_prefix(self, prefix: str, trainable: bool):
        self._check(lib().hb_paper_set_trainable_prefix(self.h, prefix.encode(), int(trainable)))

    def paper_adam_reset(self):
        self._check(lib().hb_paper_adam_reset(self.h))

    @staticmethod
    def _hist(h, n, ab):
        return TrainHistory([(i + 1, h[i, 0], h[i, 1], h[i, 2], int(h[i, 3])) for i in range(n)], bool(ab))

    def paper_train(self, cfg: TrainConfig, r_hat, e_true, model_id, kappa2, gamma) -> TrainHistory:
        """train() over an in-memory dataset (quantized samples, per-model kappa2 / gamma)"""
        r = np.ascontiguousarray(r_hat, np.float32)
        e = np.ascontiguousarray(e_true, np.float32)
        m = np.ascontiguousarray(model_id, np.int32)
        k2 = np.ascontiguousarray(kappa2, np.float64)
        g = np.ascontiguousarray(gamma, np.float64)
        N, _, H, W = r.shape
        h = np.zeros((max(cfg.epochs, 1), 4))
        n, ab = C.c_int(), C.c_int()
        c = cfg._c()
        self._check(lib().hb_paper_train(self.h, C.byref(c), N, H, W, _p(r, _fp), _p(e, _fp), _p(m, _ip), k2.shape[0],
                                         _p(k2), _p(g), _p(h), h.shape[0], C.byref(n), C.byref(ab)))
        return self._hist(h, n.value, ab.value)

    def paper_retrain(self, n_pairs: int, epochs: int, base: TrainConfig, seed: int) -> TrainHistory:
        """retrain() on this context's problem (inc/training.hpp:229-298)"""
        h = np.zeros((max(epochs, 1), 4))
        n, ab = C.c_int(), C.c_int()
        c = base._c()
        self._check(lib().hb_paper_retrain(self.h, n_pairs, epochs, C.byref(c), seed, _p(h), h.shape[0], C.byref(n),
                                           C.byref(ab)))
        return self._hist(h, n.value, ab.value)

    def encode(self):
        self._check(lib().hb_encode(self.h))

    def context_map(self, l, base=16):
        out = np.zeros((1, base, self.ny >> l, self.nx >> l), np.float32)
        self._check(lib().hb_get_context(self.h, l, _p(out, _fp)))
        return out

    # operators (inc/stencil.hpp)
    def apply(self, u, level=0, shifted=False):
        u = _c128(u)
        B = 1 if u.ndim == 2 else u.shape[0]
        y = np.zeros_like(u)
        self._check(lib().hb_operator_apply(self.h, level, int(shifted), B, _p(u), _p(y)))
        return y

    def jacobi(self, v, f, iters=1, level=0):
        v = _c128(v).copy()
        f = _c128(f)
        B = 1 if v.ndim == 2 else v.shape[0]
        self._check(lib().hb_jacobi(self.h, level, B, _p(v), _p(f), iters))
        return v

    def restrict(self, fine, level=0):
        fine = _c128(fine)
        B = 1 if fine.ndim == 2 else fine.shape[0]
        shp = fine.shape[:-2] + (fine.shape[-2] // 2, fine.shape[-1] // 2)
        out = np.zeros(shp, np.complex128)
        self._check(lib().hb_restrict(self.h, level, B, _p(fine), _p(out)))
        return out

    def prolong(self, coarse, level=0):
        coarse = _c128(coarse)
        B = 1 if coarse.ndim == 2 else coarse.shape[0]
        shp = coarse.shape[:-2] + (coarse.shape[-2] * 2, coarse.shape[-1] * 2)
        out = np.zeros(shp, np.complex128)
        self._check(lib().hb_prolong(self.h, level, B, _p(coarse), _p(out)))
        return out

    def coarse_solve(self, f):
        f = _c128(f)
        B = 1 if f.ndim == 2 else f.shape[0]
        x = np.zeros_like(f)
        self._check(lib().hb_coarse_solve(self.h, B, _p(f), _p(x)))
        return x

    def precond_apply(self, kind, r):
        r = _c128(r)
        B = 1 if r.ndim == 2 else r.shape[0]
        z = np.zeros_like(r)
        self._check(lib().hb_precond_apply(self.h, HB_PC[kind], B, _p(r), _p(z)))
        return z

    def precond_apply_device(self, kind, dr: int, dz: int, nb: int):
        """r, z: device pointers to complex64 [nb][ny][nx] (e.g. torch.complex64
        tensors' data_ptr()); enqueued on the library stream, no synchronisation."""
        self._check(lib().hb_precond_apply_device(self.h, HB_PC[kind], nb, C.c_void_p(dr), C.c_void_p(dz)))

    def fgmres(self, kind, B, cfg: KrylovConfig, X0=None, out=None):
        """out: optional preallocated (e.g. pinned) c128 array receiving X."""
        B = _c128(B)
        if B.ndim == 2:
            B = B[None]
        nb = B.shape[0]
        if out is not None:
            if out.shape != B.shape or out.dtype != np.complex128 or not out.flags.c_contiguous:
                raise ValueError("out must be a C-contiguous complex128 array shaped like B")
            X = out
        else:
            X = np.zeros_like(B)
        cap = cfg.max_iters + 2
        hist = np.zeros((nb, cap))
        hl = np.zeros(nb, np.int32)
        it = np.zeros(nb, np.int32)
        cv = np.zeros(nb, np.uint8)
        bk = np.zeros(nb, np.uint8)
        kc = _KrylovCfg(cfg.restart, cfg.max_iters, cfg.rel_tol, int(cfg.flexible))
        x0p = _p(_c128(X0)) if X0 is not None else None
        self._check(lib().hb_fgmres(self.h, C.byref(kc), HB_PC[kind], nb, _p(B), x0p, _p(X), _p(hist), cap,
                                    _p(hl, _ip), _p(it, _ip), _p(cv, _u8p), _p(bk, _u8p)))
        rep = SolveReport([hist[c, :hl[c]].copy() for c in range(nb)], [int(v) for v in it],
                          [bool(v) for v in cv], [bool(v) for v in bk])
        return X, rep

    def block_fgmres(self, kind, B, cfg: KrylovConfig, X0=None):
        """True block FGMRES (hb_block_fgmres): the columns of B share one block
        Krylov space; cfg.restart / cfg.max_iters count block steps."""
        B = _c128(B)
        if B.ndim == 2:
            B = B[None]
        nb = B.shape[0]
        X = np.zeros_like(B)
        cap = cfg.max_iters + 2
        hist = np.zeros((nb, cap))
        hl = np.zeros(nb, np.int32)
        it = np.zeros(nb, np.int32)
        cv = np.zeros(nb, np.uint8)
        bk = np.zeros(nb, np.uint8)
        kc = _KrylovCfg(cfg.restart, cfg.max_iters, cfg.rel_tol, int(cfg.flexible))
        x0p = _p(_c128(X0)) if X0 is not None else None
        self._check(lib().hb_block_fgmres(self.h, C.byref(kc), HB_PC[kind], nb, _p(B), x0p, _p(X), _p(hist), cap,
                                          _p(hl, _ip), _p(it, _ip), _p(cv, _u8p), _p(bk, _u8p)))
        rep = SolveReport([hist[c, :hl[c]].copy() for c in range(nb)], [int(v) for v in it],
                          [bool(v) for v in cv], [bool(v) for v in bk])
        return X, rep

    def gen_sample_pairs(self, seeds, k_forced=-1, k_max=10):
        """gen_sample_pair (inc/datagen.hpp:191-219) for each seed: (r, e, k) with
        r, e complex128 [count][ny][nx] and k the FGMRES iterations drawn."""
        seeds = np.ascontiguousarray(seeds, np.uint64)
        cnt = seeds.shape[0]
        r = np.zeros((cnt, self.ny, self.nx), np.complex128)
        e = np.zeros_like(r)
        k = np.zeros(cnt, np.int32)
        self._check(lib().hb_gen_sample_pairs(self.h, cnt, seeds.ctypes.data_as(C.POINTER(C.c_uint64)), k_forced,
                                              k_max, _p(r), _p(e), _p(k, _ip)))
        return r, e, k

    # ---- row slabs (one large grid over several GPUs)
    def slab_init_nccl(self, rank: int, nranks: int, nccl_id: bytes):
        """This context becomes slab `rank` of `nranks` (one GPU per process, NCCL transport)."""
        if len(nccl_id) != NCCL_ID_BYTES:
            raise ValueError("nccl_id must be 128 bytes (nccl_unique_id())")
        self._check(lib().hb_slab_init_nccl(self.h, rank, nranks, nccl_id))

    def slab_rows(self):
        lo, hi = C.c_int(), C.c_int()
        self._check(lib().hb_slab_rows(self.h, C.byref(lo), C.byref(hi)))
        return lo.value, hi.value

    def precond_apply_slab(self, kind, r):
        """M_V on this process's slab rows r [B][rows][nx] (hb_slab_rows)."""
        r = _c128(r)
        B = 1 if r.ndim == 2 else r.shape[0]
        z = np.zeros_like(r)
        self._check(lib().hb_precond_apply_slab(self.h, HB_PC[kind], B, _p(r), _p(z)))
        return z

    def fgmres_slab(self, kind, B, cfg: KrylovConfig, X0=None):
        """block_fgmres over row slabs; B, X0, X hold this process's slab rows."""
        B = _c128(B)
        if B.ndim == 2:
            B = B[None]
        nb = B.shape[0]
        X = np.zeros_like(B)
        cap = cfg.max_iters + 2
        hist = np.zeros((nb, cap))
        hl = np.zeros(nb, np.int32)
        it = np.zeros(nb, np.int32)
        cv = np.zeros(nb, np.uint8)
        bk = np.zeros(nb, np.uint8)
        kc = _KrylovCfg(cfg.restart, cfg.max_iters, cfg.rel_tol, int(cfg.flexible))
        x0p = _p(_c128(X0)) if X0 is not None else None
        self._check(lib().hb_fgmres_slab(self.h, C.byref(kc), HB_PC[kind], nb, _p(B), x0p, _p(X), _p(hist), cap,
                                         _p(hl, _ip), _p(it, _ip), _p(cv, _u8p), _p(bk, _u8p)))
        rep = SolveReport([hist[c, :hl[c]].copy() for c in range(nb)], [int(v) for v in it],
                          [bool(v) for v in cv], [bool(v) for v in bk])
        return X, rep

    def fgmres_device(self, kind, dB: int, dX: int, nb: int, cfg: KrylovConfig, want_report=True):
        """B, X are device pointers (c128 [nb][ny][nx]); e.g. torch tensors' data_ptr()."""
        kc = _KrylovCfg(cfg.restart, cfg.max_iters, cfg.rel_tol, int(cfg.flexible))
        if not want_report:
            self._check(lib().hb_fgmres_device(self.h, C.byref(kc), HB_PC[kind], nb, C.c_void_p(dB), C.c_void_p(dX),
                                               None, 0, None, None, None, None))
            return None
        cap = cfg.max_iters + 2
        hist = np.zeros((nb, cap))
        hl = np.zeros(nb, np.int32)
        it = np.zeros(nb, np.int32)
        cv = np.zeros(nb, np.uint8)
        bk = np.zeros(nb, np.uint8)
        self._check(lib().hb_fgmres_device(self.h, C.byref(kc), HB_PC[kind], nb, C.c_void_p(dB), C.c_void_p(dX),
                                           _p(hist), cap, _p(hl, _ip), _p(it, _ip), _p(cv, _u8p), _p(bk, _u8p)))
        return SolveReport([hist[c, :hl[c]].copy() for c in range(nb)], [int(v) for v in it],
                           [bool(v) for v in cv], [bool(v) for v in bk])

    def set_option(self, key: str, value: int):
        self._check(lib().hb_set_option(self.h, key.encode(), int(value)))

    # instrumentation
    def prof_enable(self, on=True):
        self._check(lib().hb_prof_enable(self.h, int(on)))

    def prof_reset(self):
        self._check(lib().hb_prof_reset(self.h))

    def prof(self):
        out = {}
        for i in range(lib().hb_prof_count(self.h)):
            ms, n, by, fl = C.c_double(), C.c_int64(), C.c_double(), C.c_double()
            self._check(lib().hb_prof_get(self.h, i, C.byref(ms), C.byref(n), C.byref(by), C.byref(fl)))
            out[lib().hb_prof_name(self.h, i).decode()] = dict(ms=ms.value, launches=n.value, bytes=by.value,
                                                               flops=fl.value)
        return out

    def prof_detail(self, on=True):
        """Switch per-launch records on/off; returns [(label, us, bytes, flops)] collected so far."""
        buf = C.create_string_buffer(1 << 22)
        self._check(lib().hb_prof_detail(self.h, int(on), buf, len(buf)))
        out = []
        for ln in buf.value.decode().splitlines():
            lab, us, by, fl = ln.rsplit(",", 3)
            out.append((lab, float(us), float(by), float(fl)))
        return out

    def launch_count(self) -> int:
        return int(lib().hb_launch_count(self.h))


# ------------------------------------------------------------ SLW1 fields
def write_slw1(path, field):
    """write_slw1 (inc/field_io.hpp:46-57): real field [ny][nx] -> f32 file."""
    f = np.ascontiguousarray(field, np.float64)
    if lib().hb_write_slw1(os.fspath(path).encode(), f.shape[1], f.shape[0], _p(f)) != 0:
        raise RuntimeError(f"cannot write {path}")


def read_slw1(path):
    """read_slw1 (inc/field_io.hpp:59-76) -> float64 [ny][nx]."""
    nx, ny = C.c_int(), C.c_int()
    p = os.fspath(path).encode()
    rc = lib().hb_read_slw1(p, C.byref(nx), C.byref(ny), None)
    if rc != 0:
        raise RuntimeError("bad SLW1 file" if rc == -4 else f"cannot open {path}")
    out = np.zeros((ny.value, nx.value))
    if lib().hb_read_slw1(p, None, None, _p(out)) != 0:
        raise RuntimeError("truncated SLW1 file")
    return out


# ------------------------------------------------------------- row slabs
NCCL_ID_BYTES = 128


def slab_partition(ny: int, levels: int, nslabs: int, slab: int):
    """Level-0 rows [begin, end) of slab `slab` (host-only; multiples of 2^(levels-1))."""
    lo, hi = C.c_int(), C.c_int()
    rc = lib().hb_slab_partition(ny, levels, nslabs, slab, C.byref(lo), C.byref(hi))
    if rc != 0:
        raise ValueError(f"no {nslabs}-slab partition of {ny} rows with {levels} levels")
    return lo.value, hi.value


def nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(NCCL_ID_BYTES)
    if lib().hb_nccl_unique_id(buf) != 0:
        raise RuntimeError("ncclGetUniqueId failed (libnccl.so.2 not loadable?)")
    return buf.raw


def slab_init_distributed(ctx: Context):
    """Slab rank = torch.distributed rank (one GPU per process): rank 0's NCCL
    unique id travels over the existing process group (plumbing only)."""
    import torch.distributed as dist
    rank, ws = dist.get_rank(), dist.get_world_size()
    obj = [nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    ctx.slab_init_nccl(rank, ws, obj[0])


def slab_init_local(ctxs: Sequence[Context]):
    """Bind contexts of this process (one device) as slabs 0..n-1; drive them through ctxs[0]."""
    arr = (_vp * len(ctxs))(*[c.h for c in ctxs])
    rc = lib().hb_slab_init_local(arr, len(ctxs))
    if rc != 0:
        msg = lib().hb_last_error(ctxs[0].h).decode()
        raise (ValueError if rc == -1 else RuntimeError)(msg)


# --------------------------------------------------------- setup helpers
def absorbing_layer(nx, ny, width, gamma_max):
    out = np.zeros((ny, nx))
    if lib().hb_absorbing_layer(nx, ny, width, gamma_max, _p(out)) != 0:
        raise ValueError("absorbing layer width out of range / gamma_max negative")
    return out


def make_medium(nx, ny, seed, sigma=8.0, vmin=1.5, vmax=4.0, n_interfaces=0, iface_seed=0, margin=16, jmin=0.5,
                jmax=1.0):
    out = np.zeros((ny, nx))
    if lib().hb_make_medium(nx, ny, seed, sigma, vmin, vmax, n_interfaces, iface_seed, margin, jmin, jmax,
                            _p(out)) != 0:
        raise ValueError("bad medium parameters")
    return out


def point_sources(seed, B, mode, lo, hi, row=0):
    xs = np.zeros(B, np.int32)
    ys = np.zeros(B, np.int32)
    lib().hb_point_sources(seed, B, mode, lo, hi, row, _p(xs, _ip), _p(ys, _ip))
    return xs, ys


def rng_normals(seed, n):
    out = np.zeros(n)
    lib().hb_rng_normals(seed, n, _p(out))
    return out


# ------------------------------------------------ reference plugin mirror
class Preconditioner:
    """inc/precond.hpp:14-27: batched apply, requires_flexible, name."""

    def apply(self, r: Sequence[np.ndarray]) -> List[np.ndarray]:
        raise NotImplementedError

    def requires_flexible(self) -> bool:
        raise NotImplementedError

    def name(self) -> str:
        raise NotImplementedError

    def apply_one(self, r):
        return self.apply([r])[0]


class _GpuPrecond(Preconditioner):
    kind = "v"

    def __init__(self, ctx: Context):
        self.ctx = ctx

    def apply(self, r):
        z = self.ctx.precond_apply(self.kind, np.stack([_c128(x) for x in r]))
        return [z[i] for i in range(z.shape[0])]

    def requires_flexible(self):
        return bool(lib().hb_precond_requires_flexible(self.ctx.h, HB_PC[self.kind]))

    def name(self):
        return lib().hb_precond_name(HB_PC[self.kind]).decode()


class SLVCyclePreconditioner(_GpuPrecond):  # M_V (inc/precond.hpp:35-53); coarse-net cycle when coarse = net
    kind = "v"


class UnetVCyclePreconditioner(_GpuPrecond):  # M_VU (inc/precond.hpp:143-165)
    kind = "vu"


class JacobiUnetPreconditioner(_GpuPrecond):  # M_JU (inc/precond.hpp:104-139), A5 net
    kind = "ju"


def check_flexible_contract(cfg: KrylovConfig, m: Preconditioner):  # inc/precond.hpp:29-32
    if m.requires_flexible() and not cfg.flexible:
        raise ValueError(f"preconditioner {m.name()} requires flexible = true")


def block_fgmres(M: _GpuPrecond, B, cfg: KrylovConfig, X0=None):
    """Device-resident block FGMRES with A = A^h of M's context (inc/krylov.hpp:83-86)."""
    check_flexible_contract(cfg, M)
    X, rep = M.ctx.fgmres(M.kind, np.stack([_c128(b) for b in B]), cfg,
                          X0=None if X0 is None else np.stack([_c128(x) for x in X0]))
    return [X[i] for i in range(X.shape[0])], rep


def convergence_factor(history, target_drop=1e6):  # inc/bench.hpp:22-38
    """(T, rho, converged): T = first t with h_t / h_0 <= 1 / target_drop, rho =
    (h_T / h_0)^(1/T); not reached -> (len - 1, nan, False).  Empty histories
    and h_0 <= 0 (or NaN) raise ValueError (std::invalid_argument, :25-26)."""
    h = np.asarray(history, dtype=np.float64)
    if h.size == 0:
        raise ValueError("empty residual history")
    if not (h[0] > 0.0):
        raise ValueError("history[0] must be positive")
    for t in range(1, len(h)):
        ratio = h[t] / h[0]
        if ratio <= 1.0 / target_drop:
            return t, ratio ** (1.0 / t), True
    return len(h) - 1, float("nan"), False
