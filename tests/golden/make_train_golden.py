"""Golden fixtures for the paper net's training, generated
by the REFERENCE ITSELF (oracle/_ref: the unmodified headers compiled in
place): traindet::run_batch + adam_step (inc/training.hpp:121-147,
inc/adam.hpp:25-58) on fixed batches, train() over a small in-memory dataset
and retrain() on one problem (inc/training.hpp:152-298).  The starting weights
are written as UNW1 checkpoints (ref_capi.cpp hr_paper_create: NetworkWeights
initialisation, seeded biases and batch-norm buffers); the trained weights too.
Run where /root/reference exists:

    bash oracle/build_ref.sh && python tests/golden/make_train_golden.py
"""
from __future__ import annotations

import math
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
from oracle import oracle as O  # noqa: E402

CFG = dict(levels=2, base=8, rpl=1, bot=1, kud=5, kres=3)
N = 16
LR = 1e-3


def problem(seed, n=N):
    om = 2 * math.pi * 1.5 * n / 10
    k2 = O.make_medium(n, n, seed)
    gam = O.absorbing_layer(n, n, 3, 2 * om)
    return k2, gam, om


def dataset(g):
    """two models x 6 quantized gen_sample_pair samples (quantize_sample, inc/datagen.hpp:290-305)"""
    r_hat, e_true, mid, k2s, gams = [], [], [], [], []
    for m, seed in enumerate((4321, 4322)):
        k2, gam, om = problem(seed)
        H = O.RefHierarchy(k2, gam, om, 1 / 16, 1 / 2.25, levels=3)
        h2 = (1.0 / N) ** 2
        for i in range(6):
            rr, ee = O.ref_gen_sample_pair(H, 900 + 10 * m + i, -1, 10)
            r_hat.append(np.stack([h2 * rr.real, h2 * rr.imag]).astype(np.float32))
            e_true.append(np.stack([ee.real, ee.imag]).astype(np.float32))
            mid.append(m)
        k2s.append(k2)
        gams.append(gam)
    g["ds_r"] = np.stack(r_hat)
    g["ds_e"] = np.stack(e_true)
    g["ds_m"] = np.asarray(mid, np.int32)
    g["ds_k2"] = np.stack(k2s)
    g["ds_gam"] = np.stack(gams)


def main():
    g = {}
    rs = np.random.default_rng(11)
    B = 3
    x = rs.standard_normal((B, 4, N, N)).astype(np.float32)
    x[:, :2] *= 0.05
    t = rs.standard_normal((B, 2, N, N)).astype(np.float32)
    kap = (0.2 + 0.5 * rs.random((B, 1, N, N))).astype(np.float32)
    g["x"], g["t"], g["kap"] = x, t, kap
    # fixed-batch steps: run_batch (train mode, gradients) + adam_step, three times
    for variant, tag in ((0, "s"), (1, "es")):
        net = O.RefPaperNet(variant=variant, seed=78, **CFG)
        net.save(os.path.join(HERE, f"train_{tag}_init.unw1"), digest=f"train-{tag}")
        k = kap if variant == 1 else None
        for step in range(3):
            loss, out, grads = net.train_batch(x, t, kappa=k, step=True, lr=LR)
            g[f"{tag}_loss{step}"] = np.float64(loss)
            if step == 0:
                g[f"{tag}_out0"], g[f"{tag}_grads0"] = out, grads
        loss, out, _ = net.train_batch(x, t, kappa=k, train_mode=False, with_grad=False)
        g[f"{tag}_eval_loss"], g[f"{tag}_eval_out"] = np.float64(loss), out
        net.save(os.path.join(HERE, f"train_{tag}_steps.unw1"), digest=f"train-{tag}-steps")
    # train(): 12 samples of two models, 3 epochs, the schedule dropping after epoch 2
    dataset(g)
    net = O.RefPaperNet(variant=0, seed=78, **CFG)
    hist, ab = net.train(3, LR, 4, 2, 0.25, False, 5, g["ds_r"], g["ds_e"], g["ds_m"], g["ds_k2"], g["ds_gam"])
    g["train_hist"], g["train_aborted"] = hist, np.int32(ab)
    net.save(os.path.join(HERE, "train_s_trained.unw1"), digest="train-s-trained")
    # retrain(): 5 fresh pairs of one problem, 2 epochs
    k2, gam, om = problem(4323)
    g["rt_k2"], g["rt_gam"], g["rt_om"] = k2, gam, np.float64(om)
    H = O.RefHierarchy(k2, gam, om, 1 / 16, 1 / 2.25, levels=3)
    for variant, tag in ((0, "s"), (1, "es")):
        net = O.RefPaperNet(variant=variant, seed=78, **CFG)
        hist, ab = net.retrain(H, 5, 2, LR, variant == 1, 17)
        g[f"rt_{tag}_hist"], g[f"rt_{tag}_aborted"] = hist, np.int32(ab)
        net.save(os.path.join(HERE, f"train_{tag}_retrained.unw1"), digest=f"retrain-{tag}")
    np.savez_compressed(os.path.join(HERE, "train.npz"), **g)
    print("wrote", sorted(g))


if __name__ == "__main__":
    main()
