"""GPU true stochastic rounding (rng=RngState) vs the reference's golden
vectors and the CPU oracle: numpy's Philox4x64-10 stream reproduced in CUDA,
every code / scale / output bit-exact."""
import json
import os

import numpy as np
import pytest
import torch

from oracle import hlq_oracle as orc

from .conftest import GOLDEN

pytestmark = pytest.mark.gpu

MANIFEST = json.load(open(os.path.join(GOLDEN, "MANIFEST.json")))
STOCH = [c for c in MANIFEST["cases"] if c.startswith("stoch")]


@pytest.fixture(scope="module")
def h():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2406_15102_b200 as h
    return h


def t(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def n(x):
    return x.detach().cpu().numpy()


def run(h, x, w, gy, rank, seed, bits_gx=4, bits_gw=8):
    plan = h.HadamardPlan(block_size=16, basis_indices=tuple(orc.lowest_sequency_bases(16, rank)))
    strat = h.BackwardStrategy("hlq", h.PathSpec("ht_quant", bits_gx), h.PathSpec("lowrank_quant", bits_gw), plan)
    rng = h.RngState(seed)
    acbp = h.acbp_compress(t(x), plan, bits=bits_gw, rng=rng)
    st = {}
    gp = h.hlq_backward(acbp, t(w), t(gy), strategy=strat, rng=rng, stages=st)
    torch.cuda.synchronize()
    return acbp, st, gp


@pytest.mark.parametrize("case", STOCH)
def test_stochastic_golden(h, case):
    g = dict(np.load(os.path.join(GOLDEN, case + ".npz")))
    acbp, st, gp = run(h, g["x"], g["w"], g["gy"], int(g["rank"]), int(g["rng_seed"]))
    assert np.array_equal(n(acbp.reference_payload()), g["x_codes"])
    assert np.array_equal(n(st["gx_codes_g"])[:, :g["gx_codes_g"].shape[1]], g["gx_codes_g"])
    assert np.array_equal(n(st["gx_codes_w"]), g["gx_codes_w"])
    assert np.array_equal(n(gp.grad_input), g["gx"])
    assert np.array_equal(n(gp.grad_weight), g["gw"])


# tokens axis with ragged L (ViT-like 197) and O; batch axis with L > 1 (index kind 2)
@pytest.mark.parametrize("B,L,I,O,rank,seed", [(3, 197, 64, 72, 8, 99), (32, 3, 16, 40, 8, 12345),
                                               (2, 64, 48, 48, 2, 2 ** 63 + 5)])
def test_stochastic_vs_oracle(h, B, L, I, O, rank, seed):
    x, w, gy = orc.make_inputs(seed % 1000, (B, L, I), (O, I), (B, L, O))
    acbp, st, gp = run(h, x, w, gy, rank, seed)
    rst = {}
    rgx, rgw = orc.hlq_backward(x, w, gy, rank=rank, stages=rst, rng=seed)
    assert np.array_equal(n(acbp.reference_payload()), rst["x_codes"])
    assert np.array_equal(n(gp.grad_input), rgx)
    assert np.array_equal(n(gp.grad_weight), rgw)


def test_stochastic_differs_from_pseudo_and_is_deterministic(h):
    x, w, gy = orc.make_inputs(3, (2, 64, 32), (48, 32), (2, 64, 48))
    _, _, a = run(h, x, w, gy, 8, 1)
    _, _, b = run(h, x, w, gy, 8, 1)
    _, _, c = run(h, x, w, gy, 8, 2)
    assert torch.equal(a.grad_input, b.grad_input) and torch.equal(a.grad_weight, b.grad_weight)
    assert not torch.equal(a.grad_input, c.grad_input)
