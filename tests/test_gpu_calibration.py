"""GPU calibrated basis selection: per-basis |coefficient|
energy of the upstream gradient on the GPU (hlq_basis_energy) vs the
reference's _basis_energy / select_bases golden outputs, and the torch-level
calibrate_bases hook."""
import json
import os

import numpy as np
import pytest
import torch

from .conftest import GOLDEN

pytestmark = pytest.mark.gpu

MANIFEST = json.load(open(os.path.join(GOLDEN, "MANIFEST.json")))
CALIB = [c for c in MANIFEST["cases"] if c.startswith("calib_")]


@pytest.fixture(scope="module")
def h():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2406_15102_b200 as h
    return h


@pytest.mark.parametrize("case", CALIB)
def test_energy_and_selection_match_reference(h, case):
    from paper_2406_15102_b200 import ops
    from paper_2406_15102_b200.backprop import _proj_view
    from paper_2406_15102_b200.hadamard import select_bases
    g = dict(np.load(os.path.join(GOLDEN, case + ".npz")))
    gy = torch.from_numpy(g["gy"]).cuda()
    B, L, O = gy.shape
    segs, rows, cols, ld, sg = _proj_view(B, L, O, int(g["axis"]))
    sums, count = ops.basis_energy(gy, segs, rows, cols, ld, sg)
    means = (sums / count).cpu().numpy()
    assert np.allclose(means, g["means"].astype(np.float64), rtol=2e-6, atol=0)
    assert select_bases(means, int(g["rank"])) == tuple(int(b) for b in g["bases"])


def test_calibrate_bases_sets_layer_plans(h):
    from paper_2406_15102_b200.layers import HLQLinear, calibrate_bases, convert_linears
    torch.manual_seed(0)
    net = convert_linears(torch.nn.Sequential(torch.nn.Linear(32, 64), torch.nn.GELU(),
                                              torch.nn.Linear(64, 16)).cuda())
    x = torch.randn(4, 48, 32, device="cuda")

    def step():
        net(x).pow(2).sum().backward()

    chosen = calibrate_bases(net, step)
    layers = [m for m in net if isinstance(m, HLQLinear)]
    assert set(chosen) == set(layers)
    for m in layers:
        assert m.strategy.plan.basis_indices == chosen[m] and len(chosen[m]) == 8
    for p in net.parameters():
        p.grad = None
    step()  # trains with the calibrated (generic bitmap) projections
    assert all(p.grad is not None and torch.isfinite(p.grad).all() for p in net.parameters())
