"""Golden fixture for the tensor-core paper U-Net (tests/test_paper_net.py::
test_paper_forward_tensor_core_sizes): UNetConfig() defaults (3 levels, base
16, 1 ResNet per level, 3 bottleneck ResNets, 5x5 down / up, 3x3 ResNets) at
128^2 -- every convolution except the 4-channel input and the 2-channel head
has channels in multiples of 16, so the device runs them as tensor-core
implicit GEMMs (5x5 stride-2 down, 3x3 ResNet, stride-2 transposed up in
parity classes).  Written by the REFERENCE ITSELF (oracle/_ref): the UNW1
checkpoint (NetworkWeights(77) + ref_capi's seeded biases / batch-norm
buffers) and the eval-mode forward of seeded inputs.

    bash oracle/build_ref.sh && python tests/golden/make_paper_tc_golden.py
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
from oracle import oracle as O  # noqa: E402

CFG = dict(levels=3, base=16, rpl=1, bot=3, kud=5, kres=3)
N = 128


def main():
    rs = np.random.default_rng(9)
    x = rs.standard_normal((2, 4, N, N)).astype(np.float32)
    net = O.RefPaperNet(variant=0, seed=77, **CFG)
    net.save(os.path.join(HERE, "paper_tc_s.unw1"), digest="golden-tc")
    y = net.forward(x)
    np.savez_compressed(os.path.join(HERE, "paper_tc.npz"), y=y)  # x: regenerated from default_rng(9)
    print("wrote paper_tc.npz", y.shape, float(np.abs(y).max()))


if __name__ == "__main__":
    main()
