"""GPU parity: the sm_100a path vs the CPU oracle / reference golden vectors.

Bar (BASELINE.json north_star): bit-exact int codes, fp32 scales and int32
accumulators; dX / dW within 1e-3 relative Frobenius -- and, with the exact
fp64 dequant epilogue used by the reference-mirroring API, bit-exact too.
Everything here goes through libhlq_b200.so (C ABI) via the package API.
"""
import json
import os

import numpy as np
import pytest
import torch

from oracle import hlq_oracle as orc

from .conftest import GOLDEN

pytestmark = pytest.mark.gpu

MANIFEST = json.load(open(os.path.join(GOLDEN, "MANIFEST.json")))
LINEAR = [c for c in MANIFEST["cases"] if c.startswith("lin")]
DEV = "cuda"


def rel_fro(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    d = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (d if d > 0 else 1.0)


def t(a, dtype=torch.float32):
    return torch.from_numpy(np.ascontiguousarray(a)).to(DEV).to(dtype)


def to_np(x):
    return x.detach().cpu().numpy()


@pytest.fixture(scope="module")
def hlq():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2406_15102_b200 as h
    from paper_2406_15102_b200 import _lib
    assert _lib.load().hlq_device_ok() == 1, "not an sm_100 device"
    return h


def _gw_codes_ref_layout(cg, axis, L, O):
    if axis == 1:
        return cg
    q = cg.shape[1]
    return cg.reshape(L, O, q).transpose(1, 2, 0).reshape(O, q * L)


def run_stages(h, x, w, gy, bases, bits_gx=4, bits_gw=8, pad_small=False):
    plan = h.HadamardPlan(block_size=16, basis_indices=tuple(int(b) for b in bases))
    strat = h.BackwardStrategy("hlq", h.PathSpec("ht_quant", bits_gx),
                               h.PathSpec("lowrank_quant", bits_gw), plan, pad_small_axes=pad_small)
    acbp = h.acbp_compress(t(x), plan, bits=bits_gw, pad_small_axes=pad_small)
    st = {}
    gp = h.hlq_backward(acbp, t(w), t(gy), strategy=strat, stages=st)
    torch.cuda.synchronize()
    B, L, O = gy.shape
    out = {k: to_np(v) for k, v in st.items() if torch.is_tensor(v)}
    out["x_codes"] = to_np(acbp.reference_payload())
    out["x_scale"] = to_np(acbp.quantized.scale)[0]
    out["axis"] = acbp.axis
    out["gw_codes_g"] = _gw_codes_ref_layout(out["gw_codes_g"], acbp.axis, L, O)
    out["gx"] = to_np(gp.grad_input)
    out["gw"] = to_np(gp.grad_weight)
    return out


def assert_stages_equal(got, ref):
    for key in ("gx_codes_g", "gx_codes_w", "x_codes", "gw_codes_g"):
        assert got[key].shape == ref[key].shape, (key, got[key].shape, ref[key].shape)
        bad = np.count_nonzero(got[key] != ref[key])
        assert bad == 0, f"{key}: {bad} codes differ"
    for key in ("gx_scale_g", "gx_scale_w", "x_scale", "gw_scale_g"):
        assert np.float32(np.asarray(got[key]).reshape(-1)[0]).tobytes() == \
            np.float32(ref[key]).tobytes(), key
    assert np.array_equal(got["gx_acc"].astype(np.int64), ref["gx_acc"]), "gx_acc"
    assert np.array_equal(got["gw_acc"].astype(np.int64), ref["gw_acc"]), "gw_acc"
    assert int(got["axis"]) == int(ref["axis"])
    assert got["gx"].shape == ref["gx"].shape and got["gw"].shape == ref["gw"].shape
    assert rel_fro(got["gx"], ref["gx"]) <= 1e-3 and rel_fro(got["gw"], ref["gw"]) <= 1e-3
    # exact fp64 epilogue: bit-identical outputs
    assert np.array_equal(got["gx"], ref["gx"]), "gx not bit-exact"
    assert np.array_equal(got["gw"], ref["gw"]), "gw not bit-exact"


@pytest.mark.parametrize("case", LINEAR)
def test_golden_linear(hlq, case):
    g = dict(np.load(os.path.join(GOLDEN, case + ".npz")))
    got = run_stages(hlq, g["x"], g["w"], g["gy"], g["bases"], int(g["bits_gx"]), int(g["bits_gw"]),
                     bool(g["pad_small"]))
    assert_stages_equal(got, g)


def oracle_stages(x, w, gy, bases, bits_gx=4, bits_gw=8, pad_small=False):
    st = {}
    gx, gw = orc.hlq_backward(x, w, gy, bases=bases, bits_gx=bits_gx, bits_gw=bits_gw,
                              pad_small_axes=pad_small, stages=st)
    st["gx"], st["gw"] = gx, gw
    return st


@pytest.mark.parametrize("shape,rank", [
    ((4096, 1, 1024, 1024), 2),   # BASELINE config (a): 2-D Linear convention, r = tokens/8
    ((4096, 1, 1024, 1024), 8),   # config (a) at the paper's default rank
    ((1, 4096, 1024, 1024), 8),   # config (a) as (1, L, I): projection along L
    ((8, 197, 768, 3072), 8),     # ViT-B/16 fc1 geometry, 8 images
    ((8, 197, 3072, 768), 8),     # ViT-B/16 fc2 geometry
    ((3, 50, 100, 1000), 4),      # ragged everything (O=1000 like a ViT head)
    ((64, 7, 40, 24), 8),         # batch axis with L > 1 (grouped K)
    ((6, 197, 128, 64), 8),       # narrow gy / x: row-grouped tiles (4 and 2 blocks per step)
    ((3, 40, 64, 32), 8),         # narrow, 8 blocks per step, ragged segments
    ((64, 7, 32, 128), 4),        # narrow on the batch axis
])
def test_seeded_vs_oracle(hlq, shape, rank):
    B, L, I, O = shape
    x, w, gy = orc.make_inputs(B * 1000 + L, (B, L, I), (O, I), (B, L, O))
    bases = orc.lowest_sequency_bases(16, rank)
    got = run_stages(hlq, x, w, gy, bases)
    ref = oracle_stages(x, w, gy, bases)
    assert_stages_equal(got, ref)


def test_bf16_inputs_match_upcast_oracle(hlq):
    B, L, I, O = 4, 197, 256, 512
    x, w, gy = orc.make_inputs(77, (B, L, I), (O, I), (B, L, O))
    xb = torch.from_numpy(x).to(torch.bfloat16)
    gb = torch.from_numpy(gy).to(torch.bfloat16)
    bases = orc.lowest_sequency_bases(16, 8)
    plan = hlq.HadamardPlan(basis_indices=bases)
    acbp = hlq.acbp_compress(xb.to(DEV), plan)
    st = {}
    gp = hlq.hlq_backward(acbp, t(w), gb.to(DEV), stages=st)
    ref = oracle_stages(xb.float().numpy(), w, gb.float().numpy(), bases)
    assert np.array_equal(to_np(acbp.reference_payload()), ref["x_codes"])
    assert np.array_equal(to_np(st["gx_codes_g"]), ref["gx_codes_g"])
    assert np.array_equal(to_np(st["gx_acc"]).astype(np.int64), ref["gx_acc"])
    assert np.array_equal(to_np(st["gw_acc"]).astype(np.int64), ref["gw_acc"])
    assert np.array_equal(to_np(gp.grad_input), ref["gx"])
    assert np.array_equal(to_np(gp.grad_weight), ref["gw"])


@pytest.mark.parametrize("m,n,k", [(128, 128, 128), (300, 200, 96), (1, 17, 16), (1000, 1000, 1008),
                                   (257, 513, 4096), (4096, 768, 3072), (3072, 768, 13312)])
def test_gemm_int_exact(hlq, m, n, k):
    from paper_2406_15102_b200 import ops
    rng = np.random.default_rng(m * 7 + n * 3 + k)
    a = rng.integers(-127, 128, size=(m, k)).astype(np.int8)
    b = rng.integers(-127, 128, size=(n, k)).astype(np.int8)
    lda = ops.pad16(k)
    A = torch.zeros((m, lda), dtype=torch.int8, device=DEV)
    Bm = torch.zeros((n, lda), dtype=torch.int8, device=DEV)
    A[:, :k] = torch.from_numpy(a).to(DEV)
    Bm[:, :k] = torch.from_numpy(b).to(DEV)
    sa = torch.tensor([0.5], device=DEV)
    sb = torch.tensor([0.25], device=DEV)
    out, acc = ops.gemm_i8(A, Bm, m, n, k, 8, 8, sa, sb, 1.0, want_acc=True)
    ref = a.astype(np.int64) @ b.astype(np.int64).T
    assert np.array_equal(to_np(acc).astype(np.int64), ref)
    assert np.array_equal(to_np(out), orc.dequant(ref, np.float32(0.5), np.float32(0.25)))


def test_int32_bound_guard(hlq):
    """Past the int32-exact bound (K * 127^2 >= 2^31) the product runs as K
    chunks summed in int64; the int32 accumulator dump is refused there, and
    K beyond the reference's MAX_K[8] = 10^6 raises ParameterError like
    int_matmul (quantize.py:19-21,166-170)."""
    from paper_2406_15102_b200 import ops
    A = torch.zeros((16, 140000), dtype=torch.int8, device=DEV)
    s = torch.ones(1, device=DEV)
    with pytest.raises(hlq.ParameterError):
        ops.gemm_i8(A, A, 16, 16, 140000, 8, 8, s, s, want_acc=True)
    big = torch.zeros((16, 1000016), dtype=torch.int8, device=DEV)
    with pytest.raises(hlq.ParameterError):
        ops.gemm_i8(big, big, 16, 16, 1000016, 8, 8, s, s)


@pytest.mark.parametrize("m,n,k,groups", [(64, 64, 200704, 1),      # ImageNet-size conv dW (K = 128*196*8)
                                          (256, 128, 140000, 1),    # just past the int32 bound
                                          (128, 64, 50176, 4)])     # grouped panels, 200,704 in total
def test_long_contraction_int64_chunks(hlq, m, n, k, groups):
    from paper_2406_15102_b200 import ops
    rng = np.random.default_rng(k + m)
    ld = ops.pad16(k)
    a = rng.integers(-127, 128, size=(groups, m, k)).astype(np.int8)
    b = rng.integers(-127, 128, size=(groups, n, k)).astype(np.int8)
    # worst case for the int32 partials: a large block of +127 * +127 products
    a[:, :, :1000] = 127
    b[:, :, :1000] = 127
    A = torch.zeros((groups, m, ld), dtype=torch.int8, device=DEV)
    Bm = torch.zeros((groups, n, ld), dtype=torch.int8, device=DEV)
    A[:, :, :k] = torch.from_numpy(a).to(DEV)
    Bm[:, :, :k] = torch.from_numpy(b).to(DEV)
    sa = torch.tensor([0.5], device=DEV)
    sb = torch.tensor([2.0 ** -20], device=DEV)
    out, _ = ops.gemm_i8(A.reshape(groups * m, ld), Bm.reshape(groups * n, ld), m, n, k, 8, 8, sa, sb, 1.0,
                         exact=True, groups=groups,
                         a_gstride=ld * m, b_gstride=ld * n)
    ref = np.zeros((m, n), dtype=np.float64)
    for g in range(groups):  # exact in fp64: every partial sum < 2^53
        ref += a[g].astype(np.float64) @ b[g].astype(np.float64).T
    assert np.abs(ref).max() * 1.0 >= 2 ** 31 or k * groups * 127 * 127 >= 2 ** 31
    assert np.array_equal(to_np(out), orc.dequant(ref.astype(np.int64), np.float32(0.5), np.float32(2.0 ** -20)))


def test_known_answers_gpu(hlq):
    c = np.load(os.path.join(GOLDEN, "ka_constant.npz"))
    a = hlq.acbp_compress(t(c["x"]), hlq.HadamardPlan())
    assert np.array_equal(to_np(a.reference_payload()), c["x_codes"])
    assert float(a.quantized.scale) == 1.0
    z = np.load(os.path.join(GOLDEN, "ka_zero.npz"))
    a = hlq.acbp_compress(t(z["x"]), hlq.HadamardPlan())
    assert float(a.quantized.scale) == 1.0 and not to_np(a.reference_payload()).any()
    assert a.payload_nbytes == 2 * 8 * 4


def test_errors_map_to_reference_classes(hlq):
    x = torch.zeros((4, 8, 16), device=DEV)
    with pytest.raises(hlq.DimensionError):
        hlq.acbp_compress(x, hlq.HadamardPlan())             # both axes < 16, no padding flag
    x = torch.randn((2, 32, 16), device=DEV)
    a = hlq.acbp_compress(x, hlq.HadamardPlan())
    with pytest.raises(hlq.StateError):
        hlq.hlq_grad_weight(a, torch.zeros((2, 16, 8), device=DEV))
    with pytest.raises(hlq.StateError):
        hlq.hlq_grad_weight(a, torch.zeros((2, 32, 8), device=DEV), bits=4)
    other = hlq.BackwardStrategy.hlq().with_plan(hlq.HadamardPlan(basis_indices=tuple(range(8))))
    with pytest.raises(hlq.StateError):
        hlq.strategy_backward(a, torch.zeros((8, 16), device=DEV), torch.zeros((2, 32, 8), device=DEV), other)
    with pytest.raises(hlq.ParameterError):
        hlq.hlq_backward(x, torch.zeros((8, 16), device=DEV), torch.zeros((2, 32, 8), device=DEV),
                         strategy=hlq.BackwardStrategy.vanilla())
    with pytest.raises(hlq.DimensionError):
        hlq.hq_grad_input(torch.zeros((2, 32, 8), device=DEV), torch.zeros((9, 16), device=DEV), 4)
    bad = torch.randn((2, 32, 16), device=DEV)
    bad[1, 3, 5] = float("inf")
    with pytest.raises(ValueError):
        hlq.acbp_compress(bad, hlq.HadamardPlan())
    with pytest.raises(hlq.ParameterError):
        hlq.acbp_compress(x, hlq.HadamardPlan(), bits=3)


def test_hlq_linear_autograd_matches_oracle(hlq):
    """HLQLinear under torch autograd: dW uses torch's 1/B-carrying dY (extra = 1),
    the fast fp32 epilogue; compare against the oracle run with extra = 1."""
    from paper_2406_15102_b200.layers import HLQLinear
    B, L, I, O = 4, 197, 384, 256
    x, w, gy = orc.make_inputs(5, (B, L, I), (O, I), (B, L, O))
    lin = HLQLinear(I, O, bias=True).to(DEV)
    with torch.no_grad():
        lin.weight.copy_(t(w))
        lin.bias.zero_()
    xt = t(x).requires_grad_(True)
    y = lin(xt)
    y.backward(t(gy))
    ref_gx, ref_gw = orc.hlq_backward(x, w, gy, rank=8, extra=1.0)
    assert rel_fro(to_np(xt.grad), ref_gx) < 1e-6
    assert rel_fro(to_np(lin.weight.grad), ref_gw) < 1e-6
    assert np.allclose(to_np(lin.bias.grad), gy.reshape(-1, O).sum(0), rtol=1e-4, atol=1e-6)

# (the bf16-autocast training path is pinned to the oracle in test_gpu_fullsize.py)


def _frac_tie_values():
    """Values v in (-0.5, 0) (scale 1) where the reference's fp32
    frac = RN(v - floor(v)) = RN(v + 1) rounds v + 1 down onto the draw
    u = bits(v) & 0x7FF / 2048 although the exact fraction exceeds it: the
    reference does NOT round up there (quantize.py:143-144).  One such value
    showed up among the 58 M gx codes of the ViT qkv layer at batch 128."""
    found = []
    for u in range(1024, 2048):
        v = np.float32((u - 2048) / 2048.0)
        for _ in range(64):
            v = np.nextafter(v, np.float32(1))
            y = np.float32(np.float32(v * np.float32(2048)) + np.float32(2048))
            if int(v.view(np.uint32) & 0x7FF) == u and float(y) == u and float(v) * 2048.0 + 2048.0 - u > 0:
                found.append(v)
                break
    vals = np.array(found, dtype=np.float32)
    # plus ordinary neighbours on both sides of zero
    rng = np.random.default_rng(3)
    extra = (rng.standard_normal(4000) * 0.3).astype(np.float32)
    return np.concatenate([vals, -vals, extra, np.float32([0.0, -0.0, -0.49999997, -1e-30])])


def test_reference_frac_rounding_ties(hlq):
    """Every quantizer entry point reproduces the reference at the fp32
    rounding of q - floor(q) for q in (-0.5, 0) (the tie cases above)."""
    from paper_2406_15102_b200 import ops
    vals = _frac_tie_values()
    assert (vals[:16] < 0).all()
    n = vals.size
    # rows of 16: [4v, 0, ..., 0] -> all 16 HT coefficients equal v; row 0 fixes amax = 7 -> scale 1
    m = np.zeros((n + 1, 16), dtype=np.float32)
    m[0, 0] = 28.0
    m[1:, 0] = 4.0 * vals
    ref_codes, ref_scale = orc.quantize(orc.transform_axis(m, 1, 16), 4)
    assert ref_scale == 1.0
    c, s, _ = ops.quant_ht_cols(t(m), 4)
    assert np.array_equal(to_np(c)[:, :16], ref_codes)
    # the same values through the projection along rows (full rank) and the batched weight codes
    mt = np.ascontiguousarray(m.T)  # (16, n+1): blocks along rows
    ref_t, _ = orc.quantize(orc.transform_axis(mt, 0, 16), 4)
    cp, k, sp, _ = ops.quant_proj_rows(t(mt), 1, 16, n + 1, 0xFFFF, 4)
    assert np.array_equal(to_np(cp)[:, :k], ref_t.T)
    (cw, sw), = ops.quant_weights([t(mt)], 4)
    assert np.array_equal(to_np(cw)[:, :16], ref_t.T)
    # dual transform of a (1, 16, n+1) gy: gx codes along cols, gw codes along rows
    g3 = np.ascontiguousarray(mt.reshape(1, 16, n + 1))
    ref_gx, _ = orc.quantize(orc.transform_axis(g3, 2, 16).reshape(16, -1), 4)
    cgx, _, cg, kg, _, _ = ops.quant_dual(t(g3), 1, 16, n + 1, 0xFFFF, 4, 8)
    assert np.array_equal(to_np(cgx)[:, :ref_gx.shape[1]], ref_gx)
    ref_gw, _ = orc.quantize(np.ascontiguousarray(orc.transform_axis(g3, 1, 16).reshape(16, -1).T), 8)
    assert np.array_equal(to_np(cg)[:, :kg], ref_gw)


@pytest.mark.parametrize("m,n,k", [(64, 27, 131072),   # ResNet CIFAR stem conv dW: split-K, N % 4 != 0
                                   (64, 27, 140000),   # ... past the int32 bound (int64 chunk sum)
                                   (100, 9, 40000)])
def test_split_k_any_n(hlq, m, n, k):
    from paper_2406_15102_b200 import ops
    rng = np.random.default_rng(m + n)
    ld = ops.pad16(k)
    a = rng.integers(-127, 128, size=(m, k)).astype(np.int8)
    b = rng.integers(-127, 128, size=(n, k)).astype(np.int8)
    A = torch.zeros((m, ld), dtype=torch.int8, device=DEV)
    Bm = torch.zeros((n, ld), dtype=torch.int8, device=DEV)
    A[:, :k] = torch.from_numpy(a).to(DEV)
    Bm[:, :k] = torch.from_numpy(b).to(DEV)
    sa = torch.tensor([0.5], device=DEV)
    sb = torch.tensor([2.0 ** -18], device=DEV)
    ref = (a.astype(np.float64) @ b.astype(np.float64).T).astype(np.int64)
    out, _ = ops.gemm_i8(A, Bm, m, n, k, 8, 8, sa, sb, 1.0, exact=True)
    assert np.array_equal(to_np(out), orc.dequant(ref, np.float32(0.5), np.float32(2.0 ** -18)))
    assert int(_lib_ws(m, n, k)) > 0  # the planner splits these long contractions


def _lib_ws(m, n, k):
    from paper_2406_15102_b200 import _lib
    return _lib.load().hlq_gemm_i8_ws_bits(m, n, k, 1, 8, 8)
