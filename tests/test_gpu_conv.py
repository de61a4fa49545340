"""GPU parity for the Conv2d lowering (reference harness/layers.py:96-158):
ACBP of im2col(x) straight from channels-last x, dW through the int8 GEMM,
dX through the int8 GEMM + col2im in the reference's tap order."""
import json
import os

import numpy as np
import pytest
import torch

from oracle import hlq_oracle as orc

from .conftest import GOLDEN

pytestmark = pytest.mark.gpu

MANIFEST = json.load(open(os.path.join(GOLDEN, "MANIFEST.json")))
CONV = [c for c in MANIFEST["cases"] if c.startswith("conv")]
DEV = "cuda"


def t(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to(DEV)


def n(x):
    return x.detach().cpu().numpy()


@pytest.fixture(scope="module")
def conv():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2406_15102_b200 import conv as c
    return c


def check(got_st, dx, dw, ref):
    for key in ("x_codes", "gx_codes_g", "gx_codes_w", "gw_codes_g"):
        g = n(got_st[key])
        assert g.shape == ref[key].shape, (key, g.shape, ref[key].shape)
        assert np.count_nonzero(g != ref[key]) == 0, key
    assert np.array_equal(n(got_st["gx_acc"]).astype(np.int64), ref["gx_acc"])
    assert np.array_equal(n(got_st["gw_acc"]).astype(np.int64), ref["gw_acc"])
    assert np.array_equal(n(dw), ref["gw"]), "dW not bit-exact"
    assert np.array_equal(n(dx), ref["gx"]), "dX not bit-exact"


@pytest.mark.parametrize("case", CONV)
def test_golden_conv(conv, case):
    g = dict(np.load(os.path.join(GOLDEN, case + ".npz")))
    st = {}
    dx, dw = conv.conv2d_hlq_backward(t(g["x"]), t(g["w"]), t(g["gy"]), int(g["stride"]), int(g["pad"]),
                                      stages=st)
    torch.cuda.synchronize()
    check(st, dx, dw, g)


@pytest.mark.parametrize("B,C,H,O,k,s,p", [
    (16, 256, 14, 256, 3, 1, 1),   # BASELINE config (b) geometry, 16 of its 128 images
    (8, 64, 32, 64, 3, 1, 1),      # ResNet-18 CIFAR stage 1 (ACBP row sharing: Wo % 16 == 0)
    (4, 128, 16, 128, 3, 1, 1),    # row sharing, 2 taps per step, one block per output row
    (2, 256, 16, 256, 3, 1, 1),    # row sharing, one tap per 256-channel step
    (2, 32, 32, 32, 5, 1, 2),      # row sharing, 5x5 (8 taps per step)
    (8, 64, 32, 128, 3, 2, 1),     # stage-2 downsampling conv
    (8, 64, 32, 128, 1, 2, 0),     # 1x1 shortcut
    (4, 3, 32, 64, 3, 1, 1),       # stem (C = 3: unaligned channel rows)
])
def test_seeded_conv_vs_oracle(conv, B, C, H, O, k, s, p):
    x, w, gy0 = orc.make_inputs(B + C + k, (B, C, H, H), (O, C, k, k), (1,))
    Ho, _ = orc.conv_out_hw(H, H, k, s, p)
    rng = np.random.default_rng(7)
    gy = (rng.lognormal(0.0, 1.4, size=(B, O, Ho, Ho)) * rng.choice([-1.0, 1.0], size=(B, O, Ho, Ho))
          * 1e-3).astype(np.float32)
    st = {}
    rst = {}
    dx, dw = conv.conv2d_hlq_backward(t(x), t(w), t(gy), s, p, stages=st)
    rdx, rdw = orc.conv2d_hlq_backward(x, w, gy, s, p, stages=rst)
    rst["gx"], rst["gw"] = rdx, rdw
    check(st, dx, dw, rst)


def test_hlq_conv2d_module_autograd(conv):
    from paper_2406_15102_b200.conv import HLQConv2d
    B, C, H, O = 8, 32, 16, 64
    x, w, _ = orc.make_inputs(3, (B, C, H, H), (O, C, 3, 3), (1,))
    rng = np.random.default_rng(4)
    gy = (rng.standard_normal((B, O, H, H)) * 1e-2).astype(np.float32)
    m = HLQConv2d(C, O, 3, padding=1, bias=True).to(DEV)
    with torch.no_grad():
        m.weight.copy_(t(w))
        m.bias.zero_()
    xt = t(x).contiguous(memory_format=torch.channels_last).requires_grad_(True)
    tf32 = torch.backends.cudnn.allow_tf32
    torch.backends.cudnn.allow_tf32 = False
    try:
        y = m(xt)
        ref_y = torch.nn.functional.conv2d(t(x), t(w), padding=1)
    finally:
        torch.backends.cudnn.allow_tf32 = tf32
    assert torch.allclose(y, ref_y, rtol=1e-4, atol=1e-4)
    y.backward(t(gy))
    rdx, rdw = orc.conv2d_hlq_backward(x, w, gy, 1, 1, extra=1.0)
    ex = np.linalg.norm(n(xt.grad) - rdx) / np.linalg.norm(rdx)
    ew = np.linalg.norm(n(m.weight.grad) - rdw) / np.linalg.norm(rdw)
    # training path: implicit-GEMM dX (taps summed in int32), fast fp32 epilogue
    assert ex < 1e-5 and ew < 1e-5, (ex, ew)
    assert np.allclose(n(m.bias.grad), gy.sum(axis=(0, 2, 3)), rtol=1e-4, atol=1e-5)


def _col2im_int(acc, B, H, W, C, k, p, Ho, Wo, s=1):
    """Integer col2im of per-tap accumulators (B*Ho*Wo, C*k*k) -> (B*H*W, C)."""
    a = acc.astype(np.int64).reshape(B, Ho, Wo, C, k, k)
    out = np.zeros((B, H + 2 * p + k * s, W + 2 * p + k * s, C), dtype=np.int64)
    for i in range(k):
        for j in range(k):
            out[:, i:i + s * (Ho - 1) + 1:s, j:j + s * (Wo - 1) + 1:s, :] += a[:, :, :, :, i, j]
    return out[:, p:p + H, p:p + W, :].reshape(B * H * W, C)


# (B, C, H, O, k, pad): 3x3 same, 1x1, valid 3x3, 5x5, O < 128 (one partial
# channel chunk), ragged O and C, M not a multiple of the 128-row tile
IMPLICIT = [
    (4, 64, 14, 256, 3, 1, 1),
    (3, 96, 9, 128, 1, 0, 1),
    (2, 48, 12, 64, 3, 0, 1),
    (2, 32, 11, 72, 5, 2, 1),
    (5, 40, 7, 200, 3, 1, 1),
    # strided: output phases (north_star item 4; ResNet downsampling convs and shortcuts)
    (4, 64, 32, 128, 3, 1, 2),   # ResNet-18 CIFAR stage-2 conv
    (4, 64, 32, 128, 1, 0, 2),   # 1x1 shortcut: three of the four phases have no tap (zero)
    (3, 48, 15, 64, 3, 1, 2),    # odd extent: phases of different sizes
    (2, 32, 13, 72, 5, 2, 2),
    (2, 40, 12, 64, 3, 0, 3),    # stride 3
]


@pytest.mark.parametrize("B,C,H,O,k,p,s", IMPLICIT)
def test_implicit_gemm_dgrad_matches_col2im(conv, B, C, H, O, k, p, s):
    from paper_2406_15102_b200.backprop import BackwardStrategy
    x, w, gy = orc.make_inputs(11 + k + p + s, (B, C, H, H), (O, C, k, k), (1,))
    Ho, _ = orc.conv_out_hw(H, H, k, s, p)
    rng = np.random.default_rng(5)
    gy = (rng.lognormal(0.0, 1.4, (B, O, Ho, Ho)) * rng.choice([-1.0, 1.0], (B, O, Ho, Ho)) * 1e-3)
    gy = gy.astype(np.float32)
    strat = BackwardStrategy.hlq()
    xt, wt, gt = t(x), t(w), t(gy)
    acbp, _ = conv.conv_acbp_compress(xt, k, s, p, strat)
    st_ref, st_imp = {}, {}
    dx_ref, _ = conv._conv_backward(acbp, wt, gt, xt.shape, s, p, strat, 1.0, True, torch.float32,
                                    need_dw=False, stages=st_ref, implicit=False)
    dx_imp, _ = conv._conv_backward(acbp, wt, gt, xt.shape, s, p, strat, 1.0, True, torch.float32,
                                    need_dw=False, stages=st_imp, implicit=True)
    torch.cuda.synchronize()
    want = _col2im_int(n(st_ref["gx_acc"]), B, H, H, C, k, p, Ho, Ho, s)
    assert np.array_equal(n(st_imp["dx_acc"]).astype(np.int64), want)
    a, b = n(dx_imp), n(dx_ref)
    assert np.linalg.norm(a - b) / np.linalg.norm(b) < 1e-6
    # and against the CPU oracle (reference Conv2d.backward, 1/B not applied to dX)
    rdx, _ = orc.conv2d_hlq_backward(x, w, gy, s, p)
    assert np.linalg.norm(a - rdx) / np.linalg.norm(rdx) < 1e-6


@pytest.mark.parametrize("B,C,H,O,k,s,p", [(4, 64, 16, 128, 3, 2, 1), (4, 64, 16, 128, 1, 2, 0),
                                           (2, 3, 32, 64, 3, 1, 1)])
def test_training_path_conv_matches_oracle(conv, B, C, H, O, k, s, p):
    """HLQConv2dFunction's training path: tap-major col2im for strided convs,
    the unfold ACBP for an RGB stem -- dW bit-for-bit the reference's codes path
    (fast epilogue: <= 1e-5), dX within fp32 rounding of the oracle."""
    from paper_2406_15102_b200.backprop import BackwardStrategy
    x, w, _ = orc.make_inputs(21 + k + s, (B, C, H, H), (O, C, k, k), (1,))
    Ho, _ = orc.conv_out_hw(H, H, k, s, p)
    rng = np.random.default_rng(9)
    gy = (rng.lognormal(0.0, 1.4, (B, O, Ho, Ho)) * rng.choice([-1.0, 1.0], (B, O, Ho, Ho)) * 1e-3)
    gy = gy.astype(np.float32)
    strat = BackwardStrategy.hlq()
    xt = t(x).contiguous(memory_format=torch.channels_last)
    acbp, _ = conv.conv_acbp_compress(xt, k, s, p, strat)
    st = {}
    acbp_ref, _ = conv.conv_acbp_compress(t(x), k, s, p, strat)
    conv._conv_backward(acbp_ref, t(w), t(gy), xt.shape, s, p, strat, 1.0, True, torch.float32, stages=st)
    assert np.array_equal(n(acbp.reference_payload()), n(acbp_ref.reference_payload()))
    dx, dw = conv._conv_backward(acbp, t(w), t(gy), xt.shape, s, p, strat, 1.0, False, torch.float32)
    rdx, rdw = orc.conv2d_hlq_backward(x, w, gy, s, p, extra=1.0)
    assert np.linalg.norm(n(dx) - rdx) / np.linalg.norm(rdx) < 1e-5
    assert np.linalg.norm(n(dw) - rdw) / np.linalg.norm(rdw) < 1e-5


def test_conv_uses_batched_weight_codes(conv):
    """HLQConv2d weight codes come from the model-wide batched refresh
    (layers.refresh_weight_codes) and give the same gradients bit for bit as
    the per-layer transform (stride 1: implicit dgrad; stride 2: GEMM + col2im)."""
    from paper_2406_15102_b200.layers import convert_linears, refresh_weight_codes
    torch.manual_seed(0)
    net = torch.nn.Sequential(torch.nn.Conv2d(16, 32, 3, padding=1), torch.nn.ReLU(),
                              torch.nn.Conv2d(32, 32, 3, stride=2, padding=1)).to(DEV)
    net = convert_linears(conv.convert_convs(net).to(memory_format=torch.channels_last))
    x = torch.randn(8, 16, 16, 16, device=DEV).to(memory_format=torch.channels_last).requires_grad_(True)

    def grads(batched):
        for m in net:
            if isinstance(m, conv.HLQConv2d):
                m._wcodes = None
        net._hlq_wcodes_hook = batched
        x.grad = None
        for p in net.parameters():
            p.grad = None
        if batched:
            assert refresh_weight_codes(net) == 2
        y = net(x) if batched else torch.nn.Sequential(*net)(x)
        y.float().square().sum().backward()
        return [x.grad.clone()] + [p.grad.clone() for p in net.parameters()]

    a = grads(True)
    assert all(m._wcodes is not None for m in net if isinstance(m, conv.HLQConv2d))
    for m in net:
        if isinstance(m, conv.HLQConv2d):
            m._wcodes = None
    b = grads(False)
    for u, v in zip(a, b):
        assert torch.equal(u, v)
