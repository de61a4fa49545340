"""Packed int4 gx codes (north_star items 1-2): the transform writes the 4-bit
dX codes two per byte, low nibble first (the ACBP container's nibble order,
acbp.py:56-61), and the dX GEMM's A path loads them packed and sign-extends
them to int8 in shared memory ahead of tcgen05 kind::i8 (no int4 MMA on
sm_100a).  Bar: the packed path's codes equal the int8 path's codes, and its
GEMM results equal the int8-operand GEMM bit for bit."""
import numpy as np
import pytest
import torch

from oracle import hlq_oracle as orc

pytestmark = pytest.mark.gpu
DEV = "cuda"


@pytest.fixture(scope="module")
def ops():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2406_15102_b200 import ops as o
    return o


@pytest.mark.parametrize("B,L,O,dtype", [(8, 197, 3072, torch.bfloat16), (3, 50, 1000, torch.float32),
                                         (4, 37, 1001, torch.float32),   # unaligned rows: fallback kernel
                                         (6, 197, 64, torch.bfloat16),   # narrow (row-grouped tiles)
                                         (128, 1, 768, torch.bfloat16)])  # batch-axis projection, L = 1
def test_packed_codes_equal_int8_codes(ops, B, L, O, dtype):
    _, _, gy = orc.make_inputs(B + L + O, (1,), (1,), (B, L, O))
    g = torch.from_numpy(gy).to(DEV).to(dtype)
    axis = 1 if L >= 16 else 0
    segs, rows, cols, ld, sg = (B, L, O, O, L * O) if axis == 1 else (1, B, L * O, L * O, B * L * O)
    a = ops.quant_dual(g, segs, rows, cols, 0x5555, 4, 8, ld, sg, colsum=True)
    p = ops.quant_dual(g, segs, rows, cols, 0x5555, 4, 8, ld, sg, colsum=True, pack_gx=True)
    assert p[0].dtype == torch.uint8 and p[0].shape[1] == ops.packed_ld(cols)
    assert torch.equal(ops.unpack_int4(p[0], ops.pad16(cols)), a[0][:, :ops.pad16(cols)])
    for i in (1, 2, 4, 6):
        assert torch.equal(p[i], a[i]), i
    # the codes are the oracle's (backprop.py:362,367)
    ref, rs = orc.quantize(orc.transform_axis(g.float().cpu().numpy(), 2, 16).reshape(B * L, -1), 4)
    assert np.array_equal(ops.unpack_int4(p[0], ops.pad16(O)).cpu().numpy(), ref)


def _codes(rng, m, k, q=7):
    return rng.integers(-q, q + 1, size=(m, k)).astype(np.int8)


def _pack(c):
    """numpy packing: byte j = (c[2j] & 0xF) | (c[2j+1] << 4)."""
    m, k = c.shape
    kk = k + (k & 1)
    cc = np.zeros((m, kk), np.int8)
    cc[:, :k] = c
    u = cc.astype(np.uint8) & 0xF
    return (u[:, 0::2] | (u[:, 1::2] << 4)).astype(np.uint8)


@pytest.mark.parametrize("m,n,k", [(128, 128, 128), (300, 200, 96), (1000, 1000, 1008), (25216, 768, 3072),
                                   (25216, 3072, 768), (4096, 768, 2304), (17, 768, 3072)])
def test_packed_gemm_equals_int8_gemm(ops, m, n, k):
    rng = np.random.default_rng(m + n + k)
    a = _codes(rng, m, k)
    b = _codes(rng, n, k)
    ld, ldp = ops.pad16(k), ops.packed_ld(k)
    A = torch.zeros((m, ld), dtype=torch.int8, device=DEV)
    A[:, :k] = torch.from_numpy(a).to(DEV)
    Bm = torch.zeros((n, ld), dtype=torch.int8, device=DEV)
    Bm[:, :k] = torch.from_numpy(b).to(DEV)
    P = torch.zeros((m, ldp), dtype=torch.uint8, device=DEV)
    pk = _pack(a)
    P[:, :pk.shape[1]] = torch.from_numpy(pk).to(DEV)
    assert torch.equal(ops.unpack_int4(P, k), A[:, :k])
    sa = torch.tensor([0.75], device=DEV)
    sb = torch.tensor([0.5], device=DEV)
    for exact, od in ((True, torch.float32), (False, torch.bfloat16)):
        ref, _ = ops.gemm_i8(A, Bm, m, n, k, 4, 4, sa, sb, 1.0, exact=exact, out_dtype=od)
        got, _ = ops.gemm_i8(P, Bm, m, n, k, 4, 4, sa, sb, 1.0, exact=exact, out_dtype=od, a_packed=True)
        assert torch.equal(got, ref), (exact, od)
    if exact:
        want = orc.dequant(a.astype(np.int64) @ b.astype(np.int64).T, np.float32(0.75), np.float32(0.5))
        got, _ = ops.gemm_i8(P, Bm, m, n, k, 4, 4, sa, sb, 1.0, exact=True, a_packed=True)
        assert np.array_equal(got.cpu().numpy(), want)


def test_pair_launch_mixed_int8_and_packed(ops):
    """The layer's dW (int8 A) and dX (packed A) in one CTA-pair launch
    (hlq_gemm_i8_multi, as HLQLinearFunction.backward runs fc1 / qkv)."""
    rng = np.random.default_rng(5)
    O, I, K, T = 3072, 768, 13312, 25216
    ga = _codes(rng, O, K, 127)
    xb = _codes(rng, I, K, 127)
    ca = _codes(rng, T, O)
    wb = _codes(rng, I, O)
    t = lambda x: torch.from_numpy(x).to(DEV)  # noqa: E731
    P = torch.zeros((T, ops.packed_ld(O)), dtype=torch.uint8, device=DEV)
    P[:, :O // 2] = t(_pack(ca))
    s = torch.tensor([0.01], device=DEV)
    assert ops.pair_eligible(O, T, K, O)
    gw, gx = ops.gemm_i8_pair(dict(a=t(ga), b=t(xb), m=O, n=I, k=K, bits_a=8, bits_b=8, sa=s, sb=s),
                              dict(a=P, b=t(wb), m=T, n=I, k=O, bits_a=4, bits_b=4, sa=s, sb=s,
                                   out_dtype=torch.bfloat16, a_packed=True))
    rw, _ = ops.gemm_i8(t(ga), t(xb), O, I, K, 8, 8, s, s, 1.0, exact=False)
    rx, _ = ops.gemm_i8(t(ca), t(wb), T, I, O, 4, 4, s, s, 1.0, exact=False, out_dtype=torch.bfloat16)
    assert torch.equal(gw, rw)
    assert torch.equal(gx, rx)
