"""Full-size parity at the BASELINE shapes, and parity of the path that trains.

* every ViT-B/16 Linear shape (qkv, proj, fc1, fc2) at batch 128, L = 197,
  through the reference-mirroring hlq_backward (backprop.py:438-447):
  codes, fp32 scales and int32 accumulators bit-exact, dX / dW bit-exact
  (exact fp64 epilogue, quantize.py:181-187);
* BASELINE config (b), Conv2d 256 -> 256, 3x3, 14x14, batch 128 (all 128
  images) through conv2d_hlq_backward (harness/layers.py:141-158);
* HLQLinear as the ViT benchmark trains it -- convert_linears (batched
  weight-codes refresh), bf16 autocast, the fused dual gy transform with the
  bias-gradient column sums, the fast epilogue, the CTA-pair GEMM launch --
  at the fc1 / fc2 shapes against the oracle fed the bf16-upcast X and dY
  with extra = 1 (torch's dY already carries 1/B, layers.py:239-250).
  Codes and scales bit-exact; dW (fp32) within 1e-3 relative Frobenius;
  dX is bf16 (x's dtype), so it is compared with the oracle's dX rounded to
  bf16, within 1e-3 relative Frobenius (the fast epilogue is <= 1 fp32 ulp
  from the exact one, so the bf16 results differ only at rounding ties).
"""
import numpy as np
import pytest
import torch

from oracle import hlq_oracle as orc

from .test_gpu_parity import assert_stages_equal, oracle_stages, rel_fro, run_stages, to_np

pytestmark = pytest.mark.gpu
DEV = "cuda"

VIT = [("qkv", 768, 2304), ("proj", 768, 768), ("fc1", 768, 3072), ("fc2", 3072, 768)]


@pytest.fixture(scope="module")
def hlq():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2406_15102_b200 as h
    from paper_2406_15102_b200 import _lib
    assert _lib.load().hlq_device_ok() == 1, "not an sm_100 device"
    return h


@pytest.mark.parametrize("name,I,O", VIT)
def test_vit_linear_batch128_bit_exact(hlq, name, I, O):
    B, L = 128, 197
    x, w, gy = orc.make_inputs(len(name) * 31 + O, (B, L, I), (O, I), (B, L, O))
    bases = orc.lowest_sequency_bases(16, 8)
    got = run_stages(hlq, x, w, gy, bases)
    ref = oracle_stages(x, w, gy, bases)
    assert_stages_equal(got, ref)


def test_conv_config_b_batch128(hlq):
    from paper_2406_15102_b200 import conv
    from .test_gpu_conv import check
    B, C, H, O, k, s, p = 128, 256, 14, 256, 3, 1, 1
    x, w, _ = orc.make_inputs(128256, (B, C, H, H), (O, C, k, k), (1,))
    rng = np.random.default_rng(17)
    gy = (rng.lognormal(0.0, 1.4, size=(B, O, H, H)) * rng.choice([-1.0, 1.0], size=(B, O, H, H))
          * 1e-3).astype(np.float32)
    st, rst = {}, {}
    dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(DEV)  # noqa: E731
    dx, dw = conv.conv2d_hlq_backward(dev(x), dev(w), dev(gy), s, p, stages=st)
    torch.cuda.synchronize()
    rdx, rdw = orc.conv2d_hlq_backward(x, w, gy, s, p, stages=rst)
    rst["gx"], rst["gw"] = rdx, rdw
    check(st, dx, dw, rst)


def _bf16_round(a: np.ndarray) -> np.ndarray:
    return torch.from_numpy(np.ascontiguousarray(a)).to(torch.bfloat16).float().numpy()


@pytest.mark.parametrize("name,I,O,packed", [("fc1", 768, 3072, False), ("fc2", 3072, 768, False),
                                            ("fc1", 768, 3072, True), ("fc2", 3072, 768, True)])
def test_training_path_autocast_vs_oracle(hlq, name, I, O, packed):
    from paper_2406_15102_b200 import layers, ops
    from paper_2406_15102_b200.layers import HLQLinear, capture_stages, convert_linears
    layers.PACK_GX[0] = packed
    B, L = 128, 197
    x, w, gy = orc.make_inputs(O * 7 + I, (B, L, I), (O, I), (B, L, O))
    net = convert_linears(torch.nn.Sequential(torch.nn.Linear(I, O))).to(DEV)
    lin = net[0]
    assert isinstance(lin, HLQLinear)
    with torch.no_grad():
        lin.weight.copy_(torch.from_numpy(w))
        lin.bias.zero_()
    xt = torch.from_numpy(x).to(DEV).requires_grad_(True)
    gyb = torch.from_numpy(gy).to(DEV).to(torch.bfloat16)
    launches0 = ops.LAUNCHES[0]
    with capture_stages() as recs:
        with torch.autocast("cuda", dtype=torch.bfloat16):
            y = net(xt)
        assert y.dtype == torch.bfloat16
        y.backward(gyb)
        torch.cuda.synchronize()
    assert lin._wcodes is not None, "batched weight-codes refresh did not run"
    assert len(recs) == 1
    layers.PACK_GX[0] = None
    st = {k: (to_np(v) if torch.is_tensor(v) else v) for k, v in recs[0].items()}
    assert st["gx_packed"] == packed
    # the oracle sees exactly the values the kernels read: bf16 X (autocast) and bf16 dY, upcast
    xb = xt.detach().to(torch.bfloat16).float().cpu().numpy()
    gb = gyb.float().cpu().numpy()
    ref = {}
    rgx, rgw = orc.hlq_backward(xb, w, gb, rank=8, extra=1.0, stages=ref)
    for key in ("gx_codes_g", "gx_codes_w", "gw_codes_g", "x_codes"):
        assert st[key].shape == ref[key].shape, (key, st[key].shape, ref[key].shape)
        bad = np.count_nonzero(st[key] != ref[key])
        assert bad == 0, f"{key}: {bad} codes differ"
    for key in ("gx_scale_g", "gx_scale_w", "gw_scale_g", "x_scale"):
        assert np.float32(np.asarray(st[key]).reshape(-1)[0]).tobytes() == np.float32(ref[key]).tobytes(), key
    assert int(st["axis"]) == int(ref["axis"])
    gx = xt.grad.float().cpu().numpy()
    assert xt.grad.dtype == torch.float32  # autocast casts x in the forward; its grad is x's dtype
    # dX went through bf16 (the layer's input dtype under autocast) before the cast back
    assert rel_fro(gx, _bf16_round(rgx)) <= 1e-3
    assert rel_fro(to_np(lin.weight.grad), rgw) <= 1e-3
    # bias gradient from the fused column sums of the bf16 dY
    gb_ref = gb.reshape(-1, O).astype(np.float64).sum(0)
    assert rel_fro(to_np(lin.bias.grad), gb_ref) <= 1e-5
    # the kernels the training path launched: ACBP, dual transform, GEMMs (+ the batched refresh)
    assert ops.LAUNCHES[0] - launches0 >= 4
