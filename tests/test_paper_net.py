"""The paper's U-Net on the GPU against the reference.

Fixtures (tests/golden/make_paper_golden.py) come from the reference itself:
UNW1 checkpoints written by its save_checkpoint, the eval-mode forward of
unet_forward / solver_forward, M_JU and M_VU applies and a 12-iteration
block_fgmres with the paper net.  Tolerances: the network computes in fp32
on both sides with different summation orders -> relative L2 1e-4 on outputs
and preconditioner applies (north_star's preconditioner bar), residual
histories 1e-3.
"""
import math
import os
import struct

import numpy as np
import pytest

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
CFG = dict(levels=3, base_channels=8, resnet_per_level=1, bottleneck_resnets=1, updown_kernel=5, res_kernel=3)
VARIANT = {"s": "standalone", "es": "encoder_solver"}


def read_unw1(path):
    """UNW1 (inc/checkpoint.hpp:12-50): [(name, dims, float32 array)], digest."""
    with open(path, "rb") as f:
        buf = f.read()
    assert buf[:4] == b"UNW1"
    ver, dl = struct.unpack_from("<II", buf, 4)
    assert ver == 1
    digest = buf[12:12 + dl].decode()
    o = 12 + dl
    (count,) = struct.unpack_from("<I", buf, o)
    o += 4
    recs = []
    for _ in range(count):
        (nl,) = struct.unpack_from("<I", buf, o)
        o += 4
        name = buf[o:o + nl].decode()
        o += nl
        dtype, rank = buf[o], buf[o + 1]
        o += 2
        assert dtype == 0 and rank == 4
        dims = struct.unpack_from("<4I", buf, o)
        o += 16
        n = int(np.prod(dims))
        recs.append((name, tuple(dims), np.frombuffer(buf, "<f4", n, o).copy()))
        o += 4 * n
    assert o == len(buf)
    return recs, digest


def test_golden_checkpoints_parse():
    """CPU: the committed reference checkpoints are well-formed UNW1 files whose
    records follow the reference's creation order (encoder first for encoder_solver)."""
    for tag in ("s", "es"):
        recs, digest = read_unw1(os.path.join(GOLD, f"paper_{tag}.unw1"))
        assert digest == f"golden-{tag}"
        names = [r[0] for r in recs]
        pre = "sol." if tag == "es" else "unet."
        if tag == "es":
            assert names[0] == "enc.entry.k" and names.index(pre + "down0.k") > names.index("enc.down2.k")
        assert names[-2:] == [pre + "out.k", pre + "out.b"]
        counts = [r[2][0] for r in recs if r[0].endswith(".count")]
        assert counts and all(c == 1.0 for c in counts)


@pytest.fixture(scope="module")
def hg():
    from paper_2203_11025_b200 import build, helmgpu
    build.build()
    return helmgpu


@pytest.fixture(scope="module")
def gold():
    return np.load(os.path.join(GOLD, "paper.npz"))


def rel(a, b):
    return float(np.linalg.norm(a - b) / (np.linalg.norm(b) + 1e-300))


def _ctx(hg, gold, tag, levels=3):
    c = hg.Context(0)
    c.set_problem(gold["k2"], gold["gamma"], float(gold["omega"]), 1 / 16, 1 / 2.25)
    c.build_hierarchy(hg.VCycleConfig(levels=levels))
    c.set_paper_net(hg.UNetConfig(**CFG), VARIANT[tag])
    c.load_checkpoint(os.path.join(GOLD, f"paper_{tag}.unw1"))
    return c


@pytest.mark.gpu
@pytest.mark.parametrize("tag", ["s", "es"])
def test_paper_registry_init_and_checkpoint_roundtrip(hg, tag, tmp_path):
    recs, _ = read_unw1(os.path.join(GOLD, f"paper_{tag}.unw1"))
    c = hg.Context(0)
    c.set_paper_net(hg.UNetConfig(**CFG), VARIANT[tag])
    assert [(n, d) for n, d in c.paper_params()] == [(n, d) for n, d, _ in recs]
    # NetworkWeights(77): every kernel drawn from the same Rng stream (the
    # fixture's biases / batch-norm buffers were re-seeded after creation)
    c.paper_init(77)
    for n, d, v in recs:
        if n.endswith((".k", ".k1", ".k2")):
            assert np.array_equal(c.paper_param(n).ravel(), v), n
    # load -> save is byte-identical (inc/checkpoint.hpp:80-82)
    c.load_checkpoint(os.path.join(GOLD, f"paper_{tag}.unw1"))
    out = tmp_path / "rt.unw1"
    c.save_checkpoint(str(out), f"golden-{tag}")
    assert out.read_bytes() == open(os.path.join(GOLD, f"paper_{tag}.unw1"), "rb").read()


@pytest.mark.gpu
@pytest.mark.parametrize("tag", ["s", "es"])
def test_paper_forward_matches_reference(hg, gold, tag):
    c = _ctx(hg, gold, tag)
    y = c.paper_forward(gold["x"])
    assert rel(y, gold[f"{tag}_y"]) < 1e-4, rel(y, gold[f"{tag}_y"])


@pytest.mark.gpu
@pytest.mark.parametrize("tag", ["s", "es"])
@pytest.mark.parametrize("kind", ["ju", "vu"])
def test_paper_preconditioners_match_reference(hg, gold, tag, kind):
    c = _ctx(hg, gold, tag)
    z = c.precond_apply(kind, gold["r"])
    assert rel(z, gold[f"{tag}_{kind}_z"]) < 1e-4, rel(z, gold[f"{tag}_{kind}_z"])


@pytest.mark.gpu
@pytest.mark.parametrize("kind", ["ju", "vu"])
def test_paper_fgmres_matches_reference(hg, gold, kind):
    """12 FGMRES(10) iterations with the standalone net made homogeneous in r
    (see make_paper_golden.py), set through the parameter API."""
    c = _ctx(hg, gold, "s")
    for name, dims in c.paper_params():
        if name.endswith((".b", ".b1", ".b2", ".offset", ".rmean")):
            c.paper_param(name, np.zeros(dims, np.float32))
        if name.endswith("out.k"):
            c.paper_param(name, c.paper_param(name) * np.float32(0.01))
    w = c.paper_param("unet.down0.k")
    w[:, 2:4] = 0.0
    c.paper_param("unet.down0.k", w)
    z0 = c.precond_apply(kind, gold["r"])
    assert rel(z0, gold[f"s_{kind}_z0"]) < 1e-4, rel(z0, gold[f"s_{kind}_z0"])
    n = gold["k2"].shape[0]
    b = np.zeros((1, n, n), np.complex128)
    b[0, n // 2, n // 3] = 1.0
    X, rep = c.fgmres(kind, b, hg.KrylovConfig(restart=10, max_iters=12))
    h, hr = rep.residual_history[0], gold[f"s_{kind}_hist"]
    assert len(h) == len(hr) and rep.iterations == [12]
    # first 6 iterations to 1e-3; M_JU then stagnates near 0.13, where the
    # complex64 Krylov basis (D0) and the fp64 reference drift apart: the
    # remaining estimates are held to 1e-2 of ||r_0||
    np.testing.assert_allclose(h[:7] / h[0], hr[:7] / hr[0], rtol=1e-3)
    assert np.max(np.abs(h / h[0] - hr / hr[0])) < 1e-2
    if kind == "vu":
        assert rel(X, gold[f"s_{kind}_X"]) < 1e-3
    else:  # stagnated: the iterate is poorly determined, its true residual is not
        res = [rel(c.apply(x), b) for x in (X, gold["s_ju_X"])]
        assert abs(res[0] - res[1]) < 2e-2, res


@pytest.mark.gpu
def test_classic_net_switches_back(hg, gold):
    """hb_set_net(slot 0) makes the classic net the network of M_JU again."""
    c = _ctx(hg, gold, "s")
    z_paper = c.precond_apply("ju", gold["r"])
    c.set_net(0, "solver", 2, 8, 3, 0)
    c.init_net_he(0, 3)
    z_classic = c.precond_apply("ju", gold["r"])
    assert rel(z_classic, z_paper) > 1e-3


@pytest.mark.gpu
def test_training_pairs_match_reference(hg, gold):
    """gen_sample_pair (inc/datagen.hpp:191-219) batched on the device: k = 0
    pins the draws bit for bit (imaginary part first, as the compiled reference
    evaluates Complex(normal(), normal())), k = 3 and the seeded random k the
    FGMRES(M_V) part; every pair satisfies A e = r (rel_residual_defect,
    :221-230, checked < 1e-10 by the reference's generator)."""
    c = hg.Context(0)
    c.set_problem(gold["k2"], gold["gamma"], float(gold["omega"]), 1 / 16, 1 / 2.25)
    c.build_hierarchy(hg.VCycleConfig(levels=3))
    r0, e0, k0 = c.gen_sample_pairs([101], k_forced=0)
    assert k0.tolist() == [0]
    assert np.array_equal(e0[0], gold["pair_101_e"])
    assert rel(r0[0], gold["pair_101_r"]) < 1e-14
    seeds = [102, 103, 104]
    r, e, k = c.gen_sample_pairs(seeds[:1], k_forced=3)
    assert rel(r[0], gold["pair_102_r"]) < 1e-4 and rel(e[0], gold["pair_102_e"]) < 1e-4
    r, e, k = c.gen_sample_pairs(seeds[1:])
    assert all(1 <= x <= 10 for x in k)
    for i, s in enumerate(seeds[1:]):
        # r is the residual of a complex64-basis iterate (D0) after k steps, so
        # its relative error grows as it shrinks: 1e-3; e = x - x~ to 1e-4
        assert rel(r[i], gold[f"pair_{s}_r"]) < 1e-3, (s, rel(r[i], gold[f"pair_{s}_r"]))
        assert rel(e[i], gold[f"pair_{s}_e"]) < 1e-4
    from oracle import oracle as O
    H = O.Hierarchy(gold["k2"], gold["gamma"], float(gold["omega"]), 1 / 16, 1 / 2.25, levels=3)
    for i in range(2):
        assert rel(H.apply(e[i]), r[i]) < 1e-10  # A e = r in fp64 (the generator's invariant)


@pytest.mark.gpu
def test_paper_forward_tensor_core_sizes(hg):
    """UNetConfig() defaults at 128^2 (tests/golden/make_paper_tc_golden.py): the
    5x5 stride-2 down convolutions, the 3x3 ResNet convolutions (bias, batch
    norm, ELU, residual add fused in the epilogue) and the stride-2 transposed
    up convolutions (four output parity classes, ELU on the inputs) run as
    3xTF32 tcgen05 implicit GEMMs (hb_conv_tc.cu); the output matches the
    reference's forward to 1e-4 and the register-tiled SIMT path to 1e-5."""
    g = np.load(os.path.join(GOLD, "paper_tc.npz"))
    x = np.random.default_rng(9).standard_normal((2, 4, 128, 128)).astype(np.float32)
    c = hg.Context(0)
    c.set_paper_net(hg.UNetConfig(levels=3, base_channels=16, resnet_per_level=1, bottleneck_resnets=3,
                                  updown_kernel=5, res_kernel=3), VARIANT["s"])
    c.load_checkpoint(os.path.join(GOLD, "paper_tc_s.unw1"))
    c.prof_enable(True)
    c.prof_detail(True)
    y = c.paper_forward(x)
    labels = [rec[0] for rec in c.prof_detail(False)]
    c.prof_enable(False)
    tc = [ln for ln in labels if ln.startswith("conv_tc")]
    assert len(tc) >= 10, labels  # down1/2, 2 x 5 ResNets, up2/up1 (the four parity classes in one GEMM)
    assert any("taps 25 s2" in ln for ln in tc) and any("par4" in ln for ln in tc), tc
    assert rel(y, g["y"]) < 1e-4, rel(y, g["y"])
    c.set_option("tconv_par4", 0)  # the transposed convs as four per-class launches
    y4 = c.paper_forward(x)
    assert rel(y, y4) < 2e-6, rel(y, y4)
    c.set_option("tc_conv", 0)
    y2 = c.paper_forward(x)
    assert rel(y, y2) < 1e-5, rel(y, y2)
    c.close()
