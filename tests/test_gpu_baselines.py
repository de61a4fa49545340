"""GPU baseline strategies (reference backprop.py:91-155,
237-347): naive int4/int8, HQ (full-rank block transform on dW), LBP-WHT
(projection + inverse projection), the bits=None float pipelines and mixed
modes, through strategy_backward on the hlq_xform kernels, vs the reference's
golden outputs.  Integer paths are bit-exact (exact epilogue); float paths use
cuBLAS fp32 GEMMs, so they match to fp32 roundoff (tolerance below)."""
import json
import os

import numpy as np
import pytest
import torch

from .conftest import GOLDEN

pytestmark = pytest.mark.gpu

MANIFEST = json.load(open(os.path.join(GOLDEN, "MANIFEST.json")))
BASELINES = [c for c in MANIFEST["cases"] if c.startswith("base_")]

# float paths: cuBLAS fp32 vs numpy fp32 summation order
RTOL, ATOL_FRAC = 1e-4, 1e-5


@pytest.fixture(scope="module")
def h():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2406_15102_b200 as h
    torch.backends.cuda.matmul.allow_tf32 = False
    return h


def _strategy(h, g):
    bits = lambda v: None if int(v) == 0 else int(v)  # noqa: E731
    plan = h.HadamardPlan(block_size=16, basis_indices=tuple(int(b) for b in g["bases"]))
    return h.BackwardStrategy(str(g["preset"]), h.PathSpec(str(g["gx_mode"]), bits(g["gx_bits"])),
                              h.PathSpec(str(g["gw_mode"]), bits(g["gw_bits"])), plan,
                              pad_small_axes=bool(g["pad_small"]))


def _close(got, ref, exact):
    got = got.detach().cpu().numpy()
    assert got.shape == ref.shape
    if exact:
        assert np.array_equal(got, ref), np.abs(got - ref).max()
    else:
        assert np.allclose(got, ref, rtol=RTOL, atol=ATOL_FRAC * float(np.abs(ref).max() + 1e-30)), \
            np.abs(got - ref).max()


@pytest.mark.parametrize("case", BASELINES)
def test_baseline_matches_reference(h, case):
    g = dict(np.load(os.path.join(GOLDEN, case + ".npz")))
    s = _strategy(h, g)
    seed = int(g["rng_seed"])
    rng = None if seed < 0 else h.RngState(seed)
    x, w, gy = (torch.from_numpy(g[k]).cuda() for k in ("x", "w", "gy"))
    gp = h.strategy_backward(x, w, gy, s, rng=rng)
    quant = lambda p: p.mode in ("quant", "ht_quant", "lowrank_quant") and p.bits is not None  # noqa: E731
    _close(gp.grad_input, g["gx"], quant(s.grad_input_path))
    _close(gp.grad_weight, g["gw"], quant(s.grad_weight_path))


def test_public_baseline_functions(h):
    g = dict(np.load(os.path.join(GOLDEN, "base_int4.npz")))
    x, w, gy = (torch.from_numpy(g[k]).cuda() for k in ("x", "w", "gy"))
    gp = h.naive_quant_backward(x, w, gy, 4)
    _close(gp.grad_input, g["gx"], True)
    _close(gp.grad_weight, g["gw"], True)
    v = dict(np.load(os.path.join(GOLDEN, "base_vanilla.npz")))
    gp = h.vanilla_backward(*(torch.from_numpy(v[k]).cuda() for k in ("x", "w", "gy")))
    _close(gp.grad_input, v["gx"], False)
    lb = dict(np.load(os.path.join(GOLDEN, "base_lbp.npz")))
    plan = h.HadamardPlan(block_size=16, basis_indices=tuple(int(b) for b in lb["bases"]))
    gp = h.lbp_wht_backward(*(torch.from_numpy(lb[k]).cuda() for k in ("x", "w", "gy")), plan)
    _close(gp.grad_input, lb["gx"], False)
    _close(gp.grad_weight, lb["gw"], False)
    with pytest.raises(h.ParameterError):
        h.lbp_wht_backward(x, w, gy, plan.with_rank(16))


@pytest.mark.parametrize("B,L,I,O", [(8, 197, 768, 256), (64, 3, 40, 72)])
def test_debug_exact_reproduces_vanilla(h, B, L, I, O):
    """debug_exact (no quantizer, full rank) must equal the plain chain rule up
    to fp32 roundoff for every strategy (test_backprop.py's degeneration check),
    at a ViT-sized token count and on the batch axis."""
    torch.manual_seed(0)
    x = torch.randn(B, L, I, device="cuda")
    w = torch.randn(O, I, device="cuda") * 0.05
    gy = torch.randn(B, L, O, device="cuda")
    ref = h.vanilla_backward(x, w, gy)
    for s in (h.BackwardStrategy.hlq(), h.BackwardStrategy.hq(), h.BackwardStrategy.lbp_wht()):
        gp = h.strategy_backward(x, w, gy, s.debug_exact())
        for got, want in ((gp.grad_input, ref.grad_input), (gp.grad_weight, ref.grad_weight)):
            err = (got - want).abs().max().item()
            assert err <= 2e-5 * want.abs().max().item(), (s.name, err)


def test_unproject_inverts_projection(h):
    """Full-rank projection followed by the inverse projection is the identity
    (orthonormal blocks), including the ragged last block."""
    from paper_2406_15102_b200.backprop import _project_f32, _unproject_f32
    torch.manual_seed(1)
    for (B, L, C), axis in (((4, 197, 96), 1), ((37, 3, 20), 0)):
        t = torch.randn(B, L, C, device="cuda")
        c = _project_f32(t, axis, 0xFFFF)
        back = _unproject_f32(c, axis, 0xFFFF, B, L, C)
        assert (back - t).abs().max().item() < 1e-5


def test_naive_quant_error_scales_with_bits(h):
    """Large-size property: the naive-quantization error of dX / dW shrinks with
    the quantizer step (int8 error a few % of the norm, int4 several times more)."""
    torch.manual_seed(2)
    B, L, I, O = 16, 197, 384, 512
    x = torch.randn(B, L, I, device="cuda")
    w = torch.randn(O, I, device="cuda") * 0.05
    gy = torch.randn(B, L, O, device="cuda")
    ref = h.vanilla_backward(x, w, gy)
    rel = {}
    for bits in (4, 8):
        gp = h.naive_quant_backward(x, w, gy, bits)
        rel[bits] = [((gp.grad_input - ref.grad_input).norm() / ref.grad_input.norm()).item(),
                     ((gp.grad_weight - ref.grad_weight).norm() / ref.grad_weight.norm()).item()]
    for i in range(2):
        assert rel[8][i] < 0.05
        assert rel[4][i] > 4 * rel[8][i]


def test_baseline_linear_module_trains(h):
    """HLQLinear under a baseline strategy routes through strategy_backward
    (raw input saved): dW equals the functional call with gw_scale = 1."""
    from paper_2406_15102_b200.layers import HLQLinear
    torch.manual_seed(3)
    lin = torch.nn.Linear(48, 40).cuda()
    for strat in (h.BackwardStrategy.naive_quant(8), h.BackwardStrategy.lbp_wht(), h.BackwardStrategy.hq()):
        m = HLQLinear.from_linear(lin, strat)
        x = torch.randn(4, 32, 48, device="cuda", requires_grad=True)
        y = m(x)
        gy = torch.randn_like(y)
        y.backward(gy)
        gp = h.strategy_backward(x.detach(), m.weight.detach(), gy, strat, gw_scale=1.0)
        assert torch.equal(m.weight.grad, gp.grad_weight)
        assert torch.equal(x.grad, gp.grad_input)
        assert torch.allclose(m.bias.grad, gy.sum((0, 1)))
