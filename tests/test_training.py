"""Training of the paper U-Net on the device against
fixtures written by the compiled reference (tests/golden/make_train_golden.py):
traindet::run_batch gradients and ADAM steps (inc/training.hpp:121-147,
inc/adam.hpp:25-58), train() and retrain() histories and trained weights
(inc/training.hpp:152-298).

Tolerances: the device sums convolutions in fp32 in another order than the
reference's sgemm, so losses and outputs of a batch are held to 1e-4 and the
gradients to 1e-3 relative L2.  Weights after ADAM steps are compared per
parameter except the biases of convolutions that feed a batch norm: their
exact gradient is zero (the batch mean removes them), both implementations
produce ~1e-9 rounding noise there, and ADAM's m / sqrt(v) turns that noise
into +-lr steps of arbitrary sign; the running means of those batch norms
track the same drift and are skipped too (the eval output, where bias and
running mean cancel, is compared).  train()/retrain() histories: 1e-3 / 2e-3
(retrain's samples come from the device gen_sample_pair, itself ~1e-4 from
the reference's).
"""
import os

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = os.path.join(HERE, "golden")
CFG = dict(levels=2, base_channels=8, resnet_per_level=1, bottleneck_resnets=1, updown_kernel=5, res_kernel=3)
LR = 1e-3


def rel(a, b):
    return float(np.linalg.norm(np.ravel(a) - np.ravel(b)) / (np.linalg.norm(np.ravel(b)) + 1e-30))


@pytest.fixture(scope="module")
def g():
    return np.load(os.path.join(GOLD, "train.npz"))


def test_golden_fixture_shapes(g):
    """CPU: the committed fixtures are complete (the GPU box has no reference)"""
    assert g["x"].shape == (3, 4, 16, 16) and g["t"].shape == (3, 2, 16, 16)
    assert g["train_hist"].shape == (3, 4) and int(g["train_aborted"]) == 0
    assert g["rt_s_hist"].shape == (2, 4) and g["rt_es_hist"].shape == (2, 4)
    for f in ("train_s_init", "train_s_steps", "train_s_trained", "train_s_retrained", "train_es_init",
              "train_es_steps", "train_es_retrained"):
        assert os.path.getsize(os.path.join(GOLD, f + ".unw1")) > 1000


def test_reference_reproduces_fixture(g):
    """CPU: the compiled reference (when present) reproduces the fixture's first
    batch bit for bit -- the fixture pins the reference, not a restatement"""
    from oracle import oracle as O
    if not O.have_ref():
        pytest.skip("oracle/_ref not built here")
    net = O.RefPaperNet(variant=0, seed=78, levels=2, base=8, rpl=1, bot=1, kud=5, kres=3)
    loss, out, grads = net.train_batch(g["x"], g["t"], step=True, lr=LR)
    assert loss == float(g["s_loss0"])
    assert np.array_equal(grads, g["s_grads0"]) and np.array_equal(out, g["s_out0"])


# ------------------------------------------------------------------ GPU ---
@pytest.fixture(scope="module")
def hg():
    from paper_2203_11025_b200 import build, helmgpu
    build.build()
    return helmgpu


def net_ctx(hg, variant, ckpt):
    ctx = hg.Context(0)
    ctx.set_paper_net(hg.UNetConfig(**CFG), variant)
    ctx.load_checkpoint(os.path.join(GOLD, ckpt))
    return ctx


def bn_fed_bias(name):
    """conv biases followed by a batch norm (down/up .b, ResNet .b1 / .b2): zero exact
    gradient; and the running means that absorb them"""
    return (name.endswith((".b", ".b1", ".b2")) and not name.endswith("out.b")) or name.endswith(".rmean")


def assert_params_match(hg, ctx, variant, ckpt, tol):
    ref = net_ctx(hg, variant, ckpt)
    worst = (0.0, "")
    for name, _ in ctx.paper_params():
        if bn_fed_bias(name):
            continue
        a, b = ctx.paper_param(name), ref.paper_param(name)
        if np.linalg.norm(b) == 0:
            assert np.linalg.norm(a) < 1e-6, name
        else:
            worst = max(worst, (rel(a, b), name))
    print("worst parameter", worst)
    assert worst[0] < tol, worst


@pytest.mark.gpu
@pytest.mark.parametrize("variant,tag", [("standalone", "s"), ("encoder_solver", "es")])
def test_train_batch_gradients_and_adam_steps(hg, g, variant, tag):
    ctx = net_ctx(hg, variant, f"train_{tag}_init.unw1")
    kap = g["kap"] if tag == "es" else None
    for step in range(3):
        loss, out = ctx.paper_train_batch(g["x"], g["t"], kappa=kap, step=True, lr=LR)
        assert abs(loss - float(g[f"{tag}_loss{step}"])) < 1e-4 * abs(float(g[f"{tag}_loss{step}"])), (step, loss)
        if step == 0:
            assert rel(out, g[f"{tag}_out0"]) < 1e-4
            gr = ctx.paper_grads()
            gref = g[f"{tag}_grads0"]
            assert gr.shape == gref.shape
            assert rel(gr, gref) < 1e-3, rel(gr, gref)
    # eval mode (running buffers updated by the three train-mode batches)
    loss, out = ctx.paper_train_batch(g["x"], g["t"], kappa=kap, train_mode=False, with_grad=False)
    assert rel(out, g[f"{tag}_eval_out"]) < 5e-3
    assert_params_match(hg, ctx, variant, f"train_{tag}_steps.unw1", 1e-5)


@pytest.mark.gpu
def test_train_loop_history_and_weights(hg, g):
    ctx = net_ctx(hg, "standalone", "train_s_init.unw1")
    cfg = hg.TrainConfig(epochs=3, lr0=LR, batch0=4, t0=2, val_fraction=0.25, seed=5)
    h = ctx.paper_train(cfg, g["ds_r"], g["ds_e"], g["ds_m"], g["ds_k2"], g["ds_gam"])
    ref = g["train_hist"]
    assert not h.aborted_non_finite and len(h.epochs) == ref.shape[0]
    got = np.array([e[1:] for e in h.epochs])
    assert np.array_equal(got[:, 2:], ref[:, 2:])  # lr, batch schedule
    np.testing.assert_allclose(got[:, :2], ref[:, :2], rtol=1e-3)
    assert_params_match(hg, ctx, "standalone", "train_s_trained.unw1", 1e-5)


@pytest.mark.gpu
@pytest.mark.parametrize("variant,tag", [("standalone", "s"), ("encoder_solver", "es")])
def test_retrain_history_and_weights(hg, g, variant, tag):
    ctx = net_ctx(hg, variant, f"train_{tag}_init.unw1")
    ctx.set_problem(g["rt_k2"], g["rt_gam"], float(g["rt_om"]), 1 / 16, 1 / 2.25)
    ctx.build_hierarchy(hg.VCycleConfig(levels=3))
    h = ctx.paper_retrain(5, 2, hg.TrainConfig(lr0=LR, encoder_solver=tag == "es"), 17)
    ref = g[f"rt_{tag}_hist"]
    got = np.array([e[1:] for e in h.epochs])
    assert got.shape == ref.shape
    np.testing.assert_allclose(got, ref, rtol=2e-3)
    assert_params_match(hg, ctx, variant, f"train_{tag}_retrained.unw1", 1e-5)


@pytest.mark.gpu
def test_train_batch_rejects_bad_input(hg):
    ctx = hg.Context(0)
    ctx.set_paper_net(hg.UNetConfig(**CFG), "standalone")
    x = np.zeros((1, 4, 18, 18), np.float32)  # not divisible by 2^levels
    with pytest.raises(Exception):
        ctx.paper_train_batch(x, np.zeros((1, 2, 18, 18), np.float32))
