"""The bf16 STATS pass with L1-bound block skipping and the input-side
min-nonzero guard (hlq_quant.cuh "bound statistics"): codes, scales, int32
accumulators and outputs must stay bit-identical to the oracle fed the
bf16-upcast inputs, on distributions chosen to stress the skip test and the
fast-division guard:

* heavy-tailed dY (SURVEY 8(d)'s lognormal(0, 1.4) * sign * 1e-3): nearly every
  block skipped once the running maximum is known;
* constant magnitude with random signs: every block's L1 equals 16c, so no
  block can be skipped against a maximum that is itself <= 16c;
* one huge outlier in the LAST row (the maximum arrives after the thresholds
  have settled on smaller blocks);
* tiny normals (1e-30) and bf16 subnormals mixed into normal data: the input
  lower bound fails the guard and the QUANT pass takes the IEEE-division path;
* a single nonzero element, and ragged L = 197 (zero-padded rows).
"""
import numpy as np
import pytest
import torch

from oracle import hlq_oracle as orc

from .test_gpu_parity import oracle_stages, to_np

pytestmark = pytest.mark.gpu
DEV = "cuda"


@pytest.fixture(scope="module")
def hlq():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2406_15102_b200 as h
    from paper_2406_15102_b200 import _lib
    assert _lib.load().hlq_device_ok() == 1, "not an sm_100 device"
    return h


def _bf16(a: np.ndarray) -> torch.Tensor:
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).to(torch.bfloat16)


def _dist(name: str, shape, seed: int) -> np.ndarray:
    rng = np.random.default_rng(seed)
    sign = rng.choice([-1.0, 1.0], size=shape)
    if name == "lognormal":
        return (rng.lognormal(0.0, 1.4, size=shape) * sign * 1e-3).astype(np.float32)
    if name == "normal":
        return (rng.standard_normal(shape) * 1e-3).astype(np.float32)
    if name == "constmag":
        return (sign * 0.375).astype(np.float32)
    if name == "outlier_last":
        a = rng.standard_normal(shape).astype(np.float32) * 1e-2
        a.reshape(-1, shape[-1])[-1, -1] = 300.0
        return a
    if name == "tiny":
        a = rng.standard_normal(shape).astype(np.float32) * 1e-3
        m = rng.random(shape) < 0.01
        a[m] = (rng.standard_normal(int(m.sum())) * 1e-30).astype(np.float32)
        return a
    if name == "subnormal":
        a = rng.standard_normal(shape).astype(np.float32)
        m = rng.random(shape) < 0.01
        a[m] = (rng.choice([-1.0, 1.0], size=int(m.sum())) * 3e-39).astype(np.float32)
        return a
    if name == "single":
        a = np.zeros(shape, dtype=np.float32)
        a.reshape(-1)[a.size // 3] = -2.5
        return a
    raise ValueError(name)


DISTS = ["lognormal", "normal", "constmag", "outlier_last", "tiny", "subnormal", "single"]


@pytest.mark.parametrize("dist", DISTS)
@pytest.mark.parametrize("shape", [(4, 197, 256, 512), (2, 64, 768, 3072)])
def test_bound_stats_bit_exact(hlq, dist, shape):
    B, L, I, O = shape
    rng = np.random.default_rng(5)
    w = (rng.standard_normal((O, I)) * (2.0 / I) ** 0.5).astype(np.float32)
    xb = _bf16(_dist(dist, (B, L, I), 11))
    gb = _bf16(_dist(dist, (B, L, O), 12))
    bases = orc.lowest_sequency_bases(16, 8)
    plan = hlq.HadamardPlan(basis_indices=bases)
    acbp = hlq.acbp_compress(xb.to(DEV), plan)
    st = {}
    gp = hlq.hlq_backward(acbp, torch.from_numpy(w).to(DEV), gb.to(DEV), stages=st)
    torch.cuda.synchronize()
    ref = oracle_stages(xb.float().numpy(), w, gb.float().numpy(), bases)
    assert np.array_equal(to_np(acbp.reference_payload()), ref["x_codes"]), "x codes"
    assert np.float32(to_np(acbp.quantized.scale)[0]).tobytes() == np.float32(ref["x_scale"]).tobytes()
    for key in ("gx_codes_g", "gx_scale_g", "gw_scale_g"):
        assert np.array_equal(np.asarray(to_np(st[key])).reshape(-1),
                              np.asarray(ref[key]).reshape(-1)), key
    assert np.array_equal(to_np(st["gx_acc"]).astype(np.int64), ref["gx_acc"])
    assert np.array_equal(to_np(st["gw_acc"]).astype(np.int64), ref["gw_acc"])
    assert np.array_equal(to_np(gp.grad_input), ref["gx"])
    assert np.array_equal(to_np(gp.grad_weight), ref["gw"])


@pytest.mark.parametrize("dist", ["lognormal", "constmag", "outlier_last", "tiny"])
def test_bound_stats_fused_dual_colsum(hlq, dist):
    """The fused dual transform as training calls it (column sums on): codes
    and scales equal the oracle's, the column sums equal the fp32 pairwise
    16-row sums accumulated over each work item and reduced in a fixed order
    (checked against an fp64 sum)."""
    from paper_2406_15102_b200 import ops
    B, L, O = 8, 197, 768
    gb = _bf16(_dist(dist, (B, L, O), 21))
    g = gb.to(DEV)
    cgx, sgx, cgw, k, sgw, _, cs = ops.quant_dual(g, B, L, O, 0x5555, 4, 8, O, L * O, colsum=True)
    torch.cuda.synchronize()
    gf = gb.float().numpy()
    ref_gx, ref_sgx = orc.quantize(orc.transform_axis(gf.reshape(B * L, O), 1, 16), 4)
    assert np.array_equal(to_np(cgx)[:, :O], ref_gx[:, :O])
    assert np.float32(to_np(sgx)[0]).tobytes() == np.float32(ref_sgx).tobytes()
    bases = orc.lowest_sequency_bases(16, 8)
    pw = orc.transform_axis(gf, 1, 16, bases)            # (B, Lp*r/16, O)
    ref_gw, ref_sgw = orc.quantize(pw, 8)
    got_gw = to_np(cgw)[:, :k].reshape(O, B, -1).transpose(1, 2, 0)
    assert np.array_equal(got_gw, ref_gw)
    assert np.float32(to_np(sgw)[0]).tobytes() == np.float32(ref_sgw).tobytes()
    ref_cs = gf.reshape(-1, O).astype(np.float64).sum(0)
    scale = np.abs(gf).reshape(-1, O).astype(np.float64).sum(0) + 1e-30
    assert np.all(np.abs(to_np(cs) - ref_cs) <= 1e-5 * scale)
