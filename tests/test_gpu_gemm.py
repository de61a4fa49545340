"""GPU: the tcgen05 int8 GEMM (both tile widths, split-K, K groups, ragged
edges) against exact int64 products on the host and the reference's fp64
dequant formula (quantize.py:152-187)."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ops():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2406_15102_b200 import _lib, ops
    assert _lib.load().hlq_device_ok() == 1
    return ops


def _ref(a, b, groups, sa, sb, extra):
    acc = np.zeros((a.shape[1], b.shape[1]), dtype=np.int64)
    for g in range(groups):
        acc += a[g].astype(np.int64) @ b[g].astype(np.int64).T
    comb = np.float64(np.float32(sa) * np.float32(sb))
    out = (acc.astype(np.float64) * (comb * np.float64(extra))).astype(np.float32)
    return acc, out


# (M, N, K, groups, bits): dX-like (many tiles), dW-like (few tiles, long K ->
# split-K), ragged M/N/K, grouped K panels, tiny
SHAPES = [
    (1000, 768, 3072, 1, 4),
    (768, 768, 13312, 1, 8),
    (3072, 768, 13312, 1, 8),
    (2304, 768, 13312, 1, 8),
    (200, 136, 4000, 1, 8),
    (130, 300, 2080, 1, 8),
    (96, 80, 48, 1, 8),
    (256, 200, 64, 9, 8),
    (384, 256, 512, 12, 8),
]


@pytest.mark.parametrize("M,N,K,groups,bits", SHAPES)
def test_gemm_exact(ops, M, N, K, groups, bits):
    rng = np.random.default_rng(M * 7 + N * 3 + K + groups)
    q = 7 if bits == 4 else 127
    ld = (K + 15) // 16 * 16
    a = np.zeros((groups, M, ld), dtype=np.int8)
    b = np.zeros((groups, N, ld), dtype=np.int8)
    a[:, :, :K] = rng.integers(-q, q + 1, (groups, M, K))
    b[:, :, :K] = rng.integers(-q, q + 1, (groups, N, K))
    sa, sb, extra = np.float32(0.0123), np.float32(3.7e-4), 1.0 / 96
    ta = torch.from_numpy(a).cuda()
    tb = torch.from_numpy(b).cuda()
    tsa = torch.tensor([sa], device="cuda")
    tsb = torch.tensor([sb], device="cuda")
    out, acc = ops.gemm_i8(ta[0] if groups == 1 else ta.view(groups * M, ld), tb[0] if groups == 1 else tb.view(groups * N, ld),
                           M, N, K, bits, bits, tsa, tsb, extra, exact=True, want_acc=True,
                           groups=groups, a_gstride=M * ld, b_gstride=N * ld)
    torch.cuda.synchronize()
    racc, rout = _ref(a[:, :, :K], b[:, :, :K], groups, sa, sb, extra)
    assert np.array_equal(acc.cpu().numpy().astype(np.int64), racc)
    assert np.array_equal(out.cpu().numpy(), rout)


def test_split_plan_used_for_dw_shapes(ops):
    from paper_2406_15102_b200 import _lib
    lib = _lib.load()
    assert lib.hlq_gemm_i8_ws(768, 768, 13312, 1) > 0        # ViT proj dW: 18 tiles
    assert lib.hlq_gemm_i8_ws(25216, 768, 3072, 1) == 0      # ViT fc1 dX: 591 tiles


def test_fast_epilogue_bf16(ops):
    rng = np.random.default_rng(5)
    M, N, K = 513, 768, 2048
    a = rng.integers(-7, 8, (M, K)).astype(np.int8)
    b = rng.integers(-7, 8, (N, K)).astype(np.int8)
    sa, sb = np.float32(0.031), np.float32(0.0007)
    out, _ = ops.gemm_i8(torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda(), M, N, K, 4, 4,
                         torch.tensor([sa], device="cuda"), torch.tensor([sb], device="cuda"), 1.0,
                         exact=False, out_dtype=torch.bfloat16)
    _, rout = _ref(a[None], b[None], 1, sa, sb, 1.0)
    got = out.float().cpu().numpy()
    assert np.linalg.norm(got - rout) / np.linalg.norm(rout) < 4e-3


def test_batched_weight_codes_match_per_tensor(ops):
    """hlq_quantize_weights (one launch for many layers) == per-tensor
    quant_proj_rows(W, 1, O, I, 0xFFFF) codes and scales, bit for bit."""
    torch.manual_seed(3)
    shapes = [(2304, 768), (768, 768), (3072, 768), (768, 3072), (1000, 768), (37, 19), (16, 1)]
    ws = [torch.randn(o, i, device="cuda") * (2.0 / i) ** 0.5 for o, i in shapes]
    ws[5][3:9] = 0.0  # zero rows inside a block
    for bits in (4, 8):
        got = ops.quant_weights(ws, bits)
        for w, (codes, scale) in zip(ws, got):
            o, i = w.shape
            ref, _, rs, _ = ops.quant_proj_rows(w, 1, o, i, 0xFFFF, bits)
            assert torch.equal(codes[:, :ops.pad16(o)], ref[:, :ops.pad16(o)])
            assert torch.equal(scale, rs)


def test_linear_uses_refreshed_weight_codes(ops):
    """The batched, cached weight codes give bit-identical gradients to the
    per-layer transform inside forward, and refresh only stale layers."""
    from paper_2406_15102_b200.layers import HLQLinear, convert_linears, refresh_weight_codes

    def make(batch):
        torch.manual_seed(7)
        net = torch.nn.Sequential(torch.nn.Linear(64, 96), torch.nn.ReLU(), torch.nn.Linear(96, 32)).cuda()
        return convert_linears(net, batch_weight_codes=batch)

    x = torch.randn(8, 20, 64, device="cuda")
    grads = []
    for batch in (True, False):
        net = make(batch)
        with torch.no_grad():
            net[0].weight.mul_(1.5)  # bump the version after construction
        xi = x.clone().requires_grad_(True)
        net(xi).sum().backward()
        layers = [m for m in net if isinstance(m, HLQLinear)]
        assert all((m.cached_weight_codes() is not None) == batch for m in layers)
        grads.append((xi.grad, net[0].weight.grad, net[2].weight.grad))
    for a, b in zip(*grads):
        assert torch.equal(a, b)
    net = make(True)
    net(x)
    with torch.no_grad():
        net[2].weight.add_(1.0)
    assert net[0].cached_weight_codes() is not None and net[2].cached_weight_codes() is None
    assert refresh_weight_codes(net) == 1


@pytest.mark.parametrize("fuse", ["1", "0"])
def test_gemm_pair_matches_separate(ops, fuse, monkeypatch):
    """A layer's dW and dX in one CTA-pair launch (LPT schedule over both
    products' tiles) == two separate fast-epilogue GEMMs, bit for bit."""
    monkeypatch.setenv("HLQ_GEMM_FUSE2", fuse)
    torch.manual_seed(4)
    O, I, T, K = 3072, 768, 4100, 2304
    cg = torch.randint(-127, 128, (O, K), dtype=torch.int8, device="cuda")
    xp = torch.randint(-127, 128, (I, K), dtype=torch.int8, device="cuda")
    cgx = torch.randint(-7, 8, (T, O), dtype=torch.int8, device="cuda")
    cw = torch.randint(-7, 8, (I, O), dtype=torch.int8, device="cuda")
    s = [torch.tensor([v], device="cuda") for v in (0.013, 0.0021, 0.37, 0.0049)]
    gw, gx = ops.gemm_i8_pair(dict(a=cg, b=xp, m=O, n=I, k=K, bits_a=8, bits_b=8, sa=s[0], sb=s[1]),
                              dict(a=cgx, b=cw, m=T, n=I, k=O, bits_a=4, bits_b=4, sa=s[2], sb=s[3],
                                   out_dtype=torch.bfloat16))
    rw, _ = ops.gemm_i8(cg, xp, O, I, K, 8, 8, s[0], s[1], 1.0, exact=False)
    rx, _ = ops.gemm_i8(cgx, cw, T, I, O, 4, 4, s[2], s[3], 1.0, exact=False, out_dtype=torch.bfloat16)
    assert torch.equal(gw, rw) and torch.equal(gx, rx)


@pytest.mark.parametrize("B,L,O,dt", [(128, 197, 768, torch.bfloat16), (4, 197, 3072, torch.bfloat16),
                                      (32, 197, 64, torch.bfloat16), (5, 40, 128, torch.float32),
                                      (64, 1, 72, torch.float32), (3, 37, 20, torch.float32),
                                      (5, 40, 36, torch.bfloat16)])
def test_dual_column_sums(ops, B, L, O, dt):
    """The bias gradient fused into the dual transform's STATS pass: fp32 column
    sums of gy (TMA path, and the plain kernel when no tensor map fits: O*2 % 16
    != 0), deterministic, codes unchanged by the extra output."""
    torch.manual_seed(0)
    gy = torch.randn(B, L, O, device="cuda").to(dt)
    segs, rows = (B, L) if L >= 16 else (1, B)
    base = ops.quant_dual(gy, segs, rows, O, 0x5555, 4, 8, O, L * O)
    r1 = ops.quant_dual(gy, segs, rows, O, 0x5555, 4, 8, O, L * O, colsum=True)
    r2 = ops.quant_dual(gy, segs, rows, O, 0x5555, 4, 8, O, L * O, colsum=True)
    ref = gy.double().reshape(-1, O).sum(0)
    assert torch.allclose(r1[6].double(), ref, rtol=1e-5, atol=1e-5 * gy.abs().max().item())
    assert torch.equal(r1[6], r2[6])  # fixed reduction order
    k = r1[3]
    assert torch.equal(r1[0], base[0]) and torch.equal(r1[2][:, :k], base[2][:, :k])
    assert torch.equal(r1[1], base[1]) and torch.equal(r1[4], base[4])


@pytest.mark.parametrize("B,L,O", [(128, 197, 3072), (128, 197, 768), (64, 1, 4096), (3, 1000, 520),
                                   (256, 256, 64), (37, 197, 128), (512, 1, 32)])
def test_fused_dynamic_transform_equals_two_static_passes(ops, B, L, O):
    """Full-size property: the fused cooperative kernel (dynamic work tickets,
    grid barrier, reversed pass 2) produces exactly the codes and scales of the
    separately launched STATS and QUANT passes (static schedule)."""
    torch.manual_seed(1)
    gy = (torch.randn(B, L, O, device="cuda") * 1e-3).to(torch.bfloat16)
    segs, rows = (B, L) if L >= 16 else (1, B)
    cgx, sgx, cgw, k, sgw, _ = ops.quant_dual(gy, segs, rows, O, 0x5555, 4, 8, O, L * O)
    st = ops.new_stats("cuda")
    ops.transform_pass(gy, segs, rows, O, O, L * O, True, True, 0x5555, 4, 8, 0, st)
    rgx = torch.empty_like(cgx)
    rgw = torch.zeros_like(cgw)
    sc = torch.empty(2, device="cuda")
    ops.transform_pass(gy, segs, rows, O, O, L * O, True, True, 0x5555, 4, 8, 1, st, rgx, rgw, sc[0:1], sc[1:2])
    assert torch.equal(sgx, sc[0:1]) and torch.equal(sgw, sc[1:2])
    assert torch.equal(cgx[:, :O], rgx[:, :O])
    assert torch.equal(cgw[:, :k], rgw[:, :k])
    x = torch.randn(B, L, O, device="cuda").to(torch.bfloat16)
    xp, kx, sx, _ = ops.quant_proj_rows(x, segs, rows, O, 0x5555, 8, O, L * O)
    st2 = ops.new_stats("cuda")
    ops.transform_pass(x, segs, rows, O, O, L * O, False, True, 0x5555, 8, 8, 0, st2)
    rx = torch.zeros_like(xp)
    ops.transform_pass(x, segs, rows, O, O, L * O, False, True, 0x5555, 8, 8, 1, st2, None, rx, None, sc[1:2])
    assert torch.equal(sx, sc[1:2]) and torch.equal(xp[:, :kx], rx[:, :kx])


def test_autocast_forward_uses_refreshed_bf16_weights(ops):
    """Under bf16 autocast the batched refresh also writes each Linear's bf16
    weight (hlq_quantize_weights_ex); the forward GEMM then uses it instead of
    a per-layer cast -- outputs and gradients bit-identical to the cast path."""
    from paper_2406_15102_b200.layers import convert_linears

    def run(batch):
        torch.manual_seed(3)
        net = convert_linears(torch.nn.Sequential(torch.nn.Linear(64, 96), torch.nn.GELU(),
                                                  torch.nn.Linear(96, 40)).cuda(), batch_weight_codes=batch)
        x = torch.randn(4, 33, 64, device="cuda", requires_grad=True)
        with torch.autocast("cuda", dtype=torch.bfloat16):
            y = net(x)
        y.float().square().sum().backward()
        if batch:
            assert net[0]._wcodes[5] is not None and net[0]._wcodes[5].dtype == torch.bfloat16
            assert torch.equal(net[0]._wcodes[5], net[0].weight.detach().to(torch.bfloat16))
        return [y.detach(), x.grad] + [p.grad for p in net.parameters()]

    for a, b in zip(run(True), run(False)):
        assert torch.equal(a, b)


def test_reserved_sms_same_results():
    """hlq_set_reserved_sms (data-parallel runs keep SMs free for NCCL): smaller
    persistent / cooperative grids, identical results."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2406_15102_b200 import _lib, ops
    lib = _lib.load()
    torch.manual_seed(0)
    gy = (torch.randn(16, 197, 3072, device="cuda") * 1e-3).to(torch.bfloat16)
    x = torch.randint(-127, 128, (768, 6656), dtype=torch.int8, device="cuda")

    def run():
        cgx, sgx, cg, k, sg, _, cs = ops.quant_dual(gy, 16, 197, 3072, 0x5555, 4, 8, 3072, 197 * 3072, colsum=True)
        w = torch.randint(-7, 8, (768, 3072), dtype=torch.int8, device="cuda")
        torch.manual_seed(1)
        dw, _ = ops.gemm_i8(cg, x, 3072, 768, k, 8, 8, sg, sg, 1.0, exact=True)
        return [cgx, sgx, cg, sg, cs, dw]
    ref = run()
    prev = lib.hlq_set_reserved_sms(40)
    try:
        got = run()
    finally:
        lib.hlq_set_reserved_sms(prev)
    for a, b in zip(ref, got):
        assert torch.equal(a, b)
