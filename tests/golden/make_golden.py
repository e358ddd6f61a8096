"""Generate tests/golden/golden.npz from the REFERENCE ITSELF: the unmodified
reference headers compiled in place (oracle/build_ref.sh -> oracle/_ref).
Run here (where /root/reference exists); the fixture is committed so the GPU
box (no /root/reference) can check against it.

    python oracle/build_ref.sh && python tests/golden/make_golden.py
"""
from __future__ import annotations

import math
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle import oracle as O  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden.npz")


def wavy(n):
    # tests/test_util.hpp:23-34 analytic kappa^2 in [0.25, 1]
    y, x = np.meshgrid(np.arange(n) / n, np.arange(n) / n, indexing="ij")
    return 0.625 + 0.3 * np.sin(3.1 * x + 1.0) * np.cos(2.3 * y)


def main():
    R = O.ref()
    g = {}
    # rng streams (inc/rng.hpp)
    u = np.zeros(16, np.uint64)
    R.hr_rng_u64(1234, 16, u.ctypes.data_as(O.C.POINTER(O.C.c_uint64)))
    g["rng_u64_1234"] = u
    nrm = np.zeros(33)
    R.hr_rng_normals(1234, 33, O._p(nrm))
    g["rng_normal_1234"] = nrm
    # absorbing layer
    a = np.zeros((32, 32))
    R.hr_absorbing_layer(32, 32, 6, 2.5, O._p(a))
    g["abl_32_6_2.5"] = a

    # wavy 16^2 problem, omega 6, abl 2 (gamma_max 0.5), 3 levels
    n = 16
    k2 = wavy(n)
    gam = np.zeros((n, n))
    R.hr_absorbing_layer(n, n, 2, 0.5, O._p(gam))
    g["wavy_k2"], g["wavy_gamma"] = k2, gam
    H = O.RefHierarchy(k2, gam, 6.0, 0.25, 1.0, levels=3)
    for l in range(3):
        k, gg, dA, dM = H.level_coef(l)
        g[f"wavy_L{l}_k2"], g[f"wavy_L{l}_gamma"], g[f"wavy_L{l}_diagA"], g[f"wavy_L{l}_diagM"] = k, gg, dA, dM
    u0 = O.random_complex_normal(7, (n, n))
    f0 = O.random_complex_normal(8, (n, n))
    g["wavy_u"], g["wavy_f"] = u0, f0
    g["wavy_Au"] = H.apply(u0)
    g["wavy_Mu"] = H.apply(u0, shifted=True)
    g["wavy_jacobi2"] = H.jacobi(u0, f0, 0.8, 2)
    for off in (0, 1):
        c = np.zeros((n // 2, n // 2), np.complex128)
        O._rcheck(R.hr_restrict(n, n, off, 2, O.cptr(u0), O.cptr(c)))
        g[f"wavy_restrict_o{off}"] = c
        fz = np.zeros((n, n), np.complex128)
        O._rcheck(R.hr_prolong(n // 2, n // 2, off, 2, O.cptr(c), O.cptr(fz)))
        g[f"wavy_prolong_o{off}"] = fz
    g["wavy_coarse_gmres_L2"] = H.coarse_gmres(O.random_complex_normal(9, (4, 4)), 2)
    g["wavy_coarse_f"] = O.random_complex_normal(9, (4, 4))
    P = O.RefPrecond("v", H)
    g["wavy_Mv_f"] = P.apply(f0)[0]

    # c0 medium at 64^2 and full size (M_V, GMRES(10) coarsest)
    for nn in (64, 128):
        om = 2 * math.pi * 1.5 * nn / 10
        k2c = O.make_medium(nn, nn, 1234)
        gc = O.absorbing_layer(nn, nn, 16, 2 * om)
        Hc = O.RefHierarchy(k2c, gc, om, 1 / 16, 1 / 2.25, levels=3)
        Pc = O.RefPrecond("v", Hc)
        b = np.zeros((1, nn, nn), np.complex128)
        b[0, nn // 2, nn // 2] = 1.0
        X, rep = O.ref_fgmres(Pc, b, restart=10, max_iters=400)
        g[f"c0_{nn}_hist"] = rep["history"][0]
        g[f"c0_{nn}_iters"] = rep["iterations"][0]
        r = O.random_complex_normal(21, (nn, nn))
        r /= np.linalg.norm(r)
        g[f"c0_{nn}_r"] = r
        g[f"c0_{nn}_Mv_r"] = Pc.apply(r)[0]
        if nn == 64:
            g["c0_64_x"] = X[0]
        g[f"c0_{nn}_k2"] = k2c

    # conv2d KAT (Tape::conv2d, im2col + GEMM)
    rng = np.random.default_rng(5)
    x = rng.standard_normal((2, 5, 12, 10)).astype(np.float32)
    w = rng.standard_normal((7, 5, 3, 3)).astype(np.float32)
    bb = rng.standard_normal(7).astype(np.float32)
    g["conv_x"], g["conv_w"], g["conv_b"], g["conv_y"] = x, w, bb, O.ref_conv2d(x, w, bb)

    # classic U-Net L=3 at 32^2 (A5/A6) and encoder-solver (A7)
    net = O.RefNet(0, 3, 16, 3, 0, seed=7)
    xi = rng.standard_normal((2, 3, 32, 32)).astype(np.float32)
    g["unet_x"], g["unet_y"] = xi, net.forward(xi)
    g["unet_w0"] = net.convs()[0][0].copy()
    enc = O.RefNet(1, 3, 16, 1, 0, seed=10)
    kap = (0.1 + 0.3 * rng.random((32, 32))).astype(np.float32)
    ctx = enc.encode(kap)
    sol = O.RefNet(0, 3, 16, 3, 16, seed=9)
    g["es_kappa"], g["es_y"] = kap, sol.forward(xi, ctx)
    for l, c in enumerate(ctx):
        g[f"es_ctx{l}"] = c

    # coarse-net 2-level cycle (A4) and M_VU (A8) at 32^2 with c0-type medium
    nn = 32
    om = 2 * math.pi * 1.5 * nn / 10
    k2c = O.make_medium(nn, nn, 1234)
    gc = O.absorbing_layer(nn, nn, 4, 2 * om)
    cnet = O.RefNet(0, 2, 16, 3, 0, seed=7)
    Hn = O.RefHierarchy(k2c, gc, om, 1 / 16, 1 / 2.25, levels=2, coarse="net", coarse_net=cnet)
    r = O.random_complex_normal(31, (nn, nn))
    r /= np.linalg.norm(r)
    g["cn_k2"], g["cn_r"] = k2c, r
    g["cn_z"] = O.RefPrecond("v", Hn).apply(r)[0]
    Hv = O.RefHierarchy(k2c, gc, om, 1 / 16, 1 / 2.25, levels=3)
    vnet = O.RefNet(0, 3, 16, 3, 0, seed=8)
    g["vu_z"] = O.RefPrecond("vu", Hv, net=vnet).apply(r)[0]
    # M_JU (inc/precond.hpp:112-130) assembled from reference primitives with the
    # classic net: e1 = J_A(0, r); de = net(h^2 (r - A e1), kappa^2); z = J_A(e1 + de, r)
    jnet = O.RefNet(0, 3, 16, 3, 0, seed=11)
    h2 = (1.0 / nn) ** 2
    e1 = Hv.jacobi(np.zeros_like(r), r, 0.8, 1, 0, shifted=False)
    res = r - Hv.apply(e1, 0, shifted=False)
    xin = np.stack([h2 * res.real, h2 * res.imag, k2c]).astype(np.float32)[None]
    de = jnet.forward(xin)[0]
    g["ju_z"] = Hv.jacobi(e1 + (de[0].astype(np.float64) + 1j * de[1].astype(np.float64)), r, 0.8, 1, 0,
                          shifted=False)
    g["ju0_z"] = Hv.jacobi(np.zeros_like(r), r, 0.8, 2, 0, shifted=False)  # zero-net M_JU == J_A o J_A

    np.savez_compressed(OUT, **g)
    print("wrote", OUT, os.path.getsize(OUT), "bytes;", len(g), "arrays")


if __name__ == "__main__":
    main()
