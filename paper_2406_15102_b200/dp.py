"""Exact data-parallel HLQ backward.

Plain DDP (bench.py) gives *replica* parity: every rank runs the reference
algorithm on its own shard with shard-local per-tensor scales, and the fp32 dW
all-reduce averages those.  That is the standard data-parallel semantics, but
it is not the single-process reference: per-tensor scales are global
quantities, and shard-local scales move dW by ~3.6 %.

This module implements *global* parity -- the sharded job reproduces the
single-process reference bit for bit:

  1. STATS pass on the local shard (hlq_transform_pass, mode 0);
  2. all-reduce(MAX) of the 4 statistics words per operand (X at forward, gy
     at backward: 2 x 16 bytes per layer) -> every rank now quantizes with the
     scale the reference computes over the whole batch;
  3. QUANT pass; int8 GEMMs produce the exact int32 dW accumulator per shard;
  4. all-reduce(SUM) of the int32 accumulators (exact, order independent --
     the same bytes as the usual fp32 dW all-reduce);
  5. one fp64 dequant, identical on every rank.
dX needs no communication (its rows are local).

Shard constraint: with the token axis as projection axis (L >= 16) any batch
split works; with the batch axis (L < 16) every shard but the last must hold
a multiple of 16 samples so no Hadamard block straddles two ranks.
"""
from __future__ import annotations

import torch
import torch.distributed as dist

from . import ops
from .backprop import BackwardStrategy, GradPair, dual_ok, ht_axis_for, _proj_view
from .errors import DimensionError, ParameterError


class Reducer:
    """The two collectives of the exact mode over a torch.distributed group."""

    def __init__(self, group=None):
        self.group = group

    def max_stats(self, stats: torch.Tensor) -> torch.Tensor:
        """Element-wise UNSIGNED max of uint32 statistics words (int32 storage)
        across ranks; reduced in int64 so words >= 2^31 order correctly."""
        wide = stats.to(torch.int64) & 0xFFFFFFFF
        dist.all_reduce(wide, op=dist.ReduceOp.MAX, group=self.group)
        out = (wide & 0xFFFFFFFF)
        out = torch.where(out >= 2 ** 31, out - 2 ** 32, out).to(torch.int32)
        stats.copy_(out)
        return stats

    def sum_acc(self, acc: torch.Tensor) -> torch.Tensor:
        dist.all_reduce(acc, op=dist.ReduceOp.SUM, group=self.group)
        return acc


class ExactDP:
    """The exact (global-scale) data-parallel mode of the HLQ autograd modules.

    Attached to every HLQLinear of a model by enable_exact_dp(); the layer's
    forward ACBP and backward gy transform then run as STATS pass ->
    all-reduce(MAX) of the 16-byte statistics -> QUANT pass, so every rank
    quantizes with the scale the single-process reference computes over the
    whole batch (quantize.py:94-100), and dW is the all-reduce(SUM) of the
    exact int32 accumulators followed by one dequant (backprop.py:407-410).
    The accumulator all-reduce is asynchronous: the layer's dX GEMM (local
    rows, no communication) runs under it.  dW comes back already averaged
    over ranks (torch's mean-loss convention), so the HLQ weights are excluded
    from DDP; every other parameter stays with DDP."""

    def __init__(self, group=None):
        self.group = group
        self.reducer = Reducer(group)
        self.world = dist.get_world_size(group)

    def quant_rows(self, src, segs, rows, cols, ld_src, seg_src, bitmap, bits):
        """Global-scale projection along rows (the ACBP of X): codes (cols, pad16(K)), K, scale."""
        dev = src.device
        st = ops.new_stats(dev)
        ops.transform_pass(src, segs, rows, cols, ld_src, seg_src, False, True, bitmap, bits, bits, 0, st)
        self.reducer.max_stats(st)
        k = ops.proj_rows_k(segs, rows, bin(bitmap).count("1"))
        codes = torch.empty((cols, max(ops.pad16(k), 16)), dtype=torch.int8, device=dev)
        scale = torch.empty(1, dtype=torch.float32, device=dev)
        ops.transform_pass(src, segs, rows, cols, ld_src, seg_src, False, True, bitmap, bits, bits, 1, st,
                           dst_gw=codes, scale_gw=scale)
        return codes, k, scale

    def quant_conv(self, x_nhwc, k, stride, pad, bitmap, bits):
        """Global-scale ACBP of im2col(x) (the conv input, channels-last):
        codes (C*k*k, pad16(K)), K, scale."""
        B, H, W, C = x_nhwc.shape
        Ho, Wo = ops.conv_out_hw(H, W, k, stride, pad)
        kk = B * ((Ho * Wo + 15) // 16) * bin(bitmap).count("1")
        st = ops.new_stats(x_nhwc.device)
        ops.conv_acbp_pass(x_nhwc, k, stride, pad, bitmap, bits, 0, st)
        self.reducer.max_stats(st)
        codes = torch.empty((C * k * k, max(ops.pad16(kk), 16)), dtype=torch.int8, device=x_nhwc.device)
        scale = torch.empty(1, dtype=torch.float32, device=x_nhwc.device)
        ops.conv_acbp_pass(x_nhwc, k, stride, pad, bitmap, bits, 1, st, codes, scale)
        return codes, kk, scale

    def quant_gy(self, gy3, axis, bitmap, bits_gx, bits_gw):
        """Both gy operands with global scales: (gx codes (T, pad16(O)), gx scale,
        gw codes (O, pad16(K)), K, gw scale)."""
        B, L, O = gy3.shape
        dev = gy3.device
        segs, rows, cols, ld, sg = _proj_view(B, L, O, axis)
        k = ops.proj_rows_k(segs, rows, bin(bitmap).count("1"))
        cgx = torch.empty((B * L, ops.pad16(O)), dtype=torch.int8, device=dev)
        cgw = torch.empty((cols, max(ops.pad16(k), 16)), dtype=torch.int8, device=dev)
        scales = torch.empty(2, dtype=torch.float32, device=dev)
        st = ops.new_stats(dev)
        dual = dual_ok(B, L, axis)
        if dual:
            ops.transform_pass(gy3, segs, rows, cols, ld, sg, True, True, bitmap, bits_gx, bits_gw, 0, st)
        else:
            ops.transform_pass(gy3, 1, B * L, O, O, B * L * O, True, False, 0xFFFF, bits_gx, bits_gx, 0, st)
            ops.transform_pass(gy3, segs, rows, cols, ld, sg, False, True, bitmap, bits_gw, bits_gw, 0, st)
        self.reducer.max_stats(st)
        if dual:
            ops.transform_pass(gy3, segs, rows, cols, ld, sg, True, True, bitmap, bits_gx, bits_gw, 1, st,
                               dst_gx=cgx, dst_gw=cgw, scale_gx=scales[0:1], scale_gw=scales[1:2])
        else:
            ops.transform_pass(gy3, 1, B * L, O, O, B * L * O, True, False, 0xFFFF, bits_gx, bits_gx, 1, st,
                               dst_gx=cgx, scale_gx=scales[0:1])
            ops.transform_pass(gy3, segs, rows, cols, ld, sg, False, True, bitmap, bits_gw, bits_gw, 1, st,
                               dst_gw=cgw, scale_gw=scales[1:2])
        return cgx, scales[0:1], cgw, k, scales[1:2]

    def reduce_acc_async(self, acc: torch.Tensor, k_local: int, groups: int, bits: int):
        """Start the all-reduce(SUM) of the int32 dW accumulator; widened to
        int64 when the global contraction could overflow int32.  Returns
        (tensor being reduced, work handle)."""
        qmax = (1 << (bits - 1)) - 1
        if k_local * groups * self.world * qmax * qmax >= 2 ** 31:
            acc = acc.to(torch.int64)
        work = dist.all_reduce(acc, op=dist.ReduceOp.SUM, group=self.group, async_op=True)
        return acc, work

    def dequant_fast(self, acc, sa, sb, out_dtype=torch.float32):
        """The GEMM's fast epilogue on the summed accumulator:
        f32(acc) * f32(f64(f32(sa*sb)) / world)  (1/world: torch's mean over ranks)."""
        scale = ((sa.float() * sb.float()).to(torch.float64) * (1.0 / self.world)).to(torch.float32)
        return (acc.to(torch.float32) * scale).to(out_dtype)


def enable_exact_dp(model: torch.nn.Module, group=None):
    """Switch every HLQLinear / HLQConv2d under `model` to the exact data-parallel mode
    and return the parameter names DDP must ignore (their gradients are
    all-reduced inside the layers):

        names = enable_exact_dp(model)
        DistributedDataParallel._set_params_and_buffers_to_ignore_for_model(model, names)
        model = DistributedDataParallel(model, ...)
    """
    from .conv import HLQConv2d
    from .layers import HLQLinear
    dp = ExactDP(group)
    names = []
    for name, m in model.named_modules():
        if isinstance(m, (HLQLinear, HLQConv2d)):
            m.dp = dp
            names.append(f"{name}.weight" if name else "weight")
    return names


def dequant(acc: torch.Tensor, sa: torch.Tensor, sb: torch.Tensor, extra: float) -> torch.Tensor:
    """out = f32(f64(acc) * (f64(f32(sa * sb)) * extra)) -- quantize.py:181-187."""
    comb = (sa.float() * sb.float()).to(torch.float64)
    return (acc.to(torch.float64) * (comb * float(extra))).to(torch.float32)


def hlq_backward_global(x: torch.Tensor, w: torch.Tensor, gy: torch.Tensor, batch_global: int,
                        reducer: Reducer, strategy: BackwardStrategy | None = None) -> GradPair:
    """HLQ backward of one Linear layer on this rank's batch shard with the
    exact global scales.  x (b, L, I) / gy (b, L, O) are the local shard;
    returns (local dX rows, global dW) -- dW equal on every rank and bit-equal
    to the single-process reference (backprop.py:438-447, extra = 1/B)."""
    strategy = strategy or BackwardStrategy.hlq()
    if x.dim() != 3 or gy.dim() != 3 or w.dim() != 2:
        raise DimensionError("expected x (b,L,I), w (O,I), gy (b,L,O)")
    b, L, I = x.shape
    O = w.shape[0]
    plan = strategy.plan
    bitmap = plan.gpu_bitmap()
    bits_gx = strategy.grad_input_path.bits or 4
    bits_gw = strategy.grad_weight_path.bits or 8
    axis = ht_axis_for(batch_global, L, plan.block_size, strategy.pad_small_axes)
    if axis == 0 and b % 16 and dist.get_rank(self_group(reducer)) != dist.get_world_size(self_group(reducer)) - 1:
        raise ParameterError("batch-axis projection: every shard but the last needs a multiple of 16 samples")
    dev = x.device
    # ---- X (ACBP): global stats, then codes
    sx_stats = ops.new_stats(dev)
    segs, rows, cols, ld, sg = _proj_view(b, L, I, axis)
    ops.transform_pass(x, segs, rows, cols, ld, sg, False, True, bitmap, bits_gw, bits_gw, 0, sx_stats)
    reducer.max_stats(sx_stats)
    k = ops.proj_rows_k(segs, rows, plan.rank)
    ldk = max(ops.pad16(k), 16)
    xp = torch.empty((cols, ldk), dtype=torch.int8, device=dev)
    scales = torch.empty(4, dtype=torch.float32, device=dev)  # x, gx, gw, w
    ops.transform_pass(x, segs, rows, cols, ld, sg, False, True, bitmap, bits_gw, bits_gw, 1, sx_stats,
                       dst_gw=xp, scale_gw=scales[0:1])
    # ---- gy: both operands, global stats, then codes
    g_stats = ops.new_stats(dev)
    segs, rows, cols, ld, sg = _proj_view(b, L, O, axis)
    cgx = torch.empty((b * L, ops.pad16(O)), dtype=torch.int8, device=dev)
    cgw = torch.empty((cols, ldk), dtype=torch.int8, device=dev)
    if dual_ok(b, L, axis):
        ops.transform_pass(gy, segs, rows, cols, ld, sg, True, True, bitmap, bits_gx, bits_gw, 0, g_stats)
    else:
        ops.transform_pass(gy, 1, b * L, O, O, b * L * O, True, False, 0xFFFF, bits_gx, bits_gx, 0, g_stats)
        ops.transform_pass(gy, segs, rows, cols, ld, sg, False, True, bitmap, bits_gw, bits_gw, 0, g_stats)
    reducer.max_stats(g_stats)
    if dual_ok(b, L, axis):
        ops.transform_pass(gy, segs, rows, cols, ld, sg, True, True, bitmap, bits_gx, bits_gw, 1, g_stats,
                           dst_gx=cgx, dst_gw=cgw, scale_gx=scales[1:2], scale_gw=scales[2:3])
    else:
        ops.transform_pass(gy, 1, b * L, O, O, b * L * O, True, False, 0xFFFF, bits_gx, bits_gx, 1,
                           g_stats, dst_gx=cgx, scale_gx=scales[1:2])
        ops.transform_pass(gy, segs, rows, cols, ld, sg, False, True, bitmap, bits_gw, bits_gw, 1,
                           g_stats, dst_gw=cgw, scale_gw=scales[2:3])
    # ---- dW: exact int32 partial sums, all-reduced, one dequant
    groups = L if axis == 0 else 1
    _, acc = ops.gemm_i8(cgw, xp, O, I, k, bits_gw, bits_gw, scales[2:3], scales[0:1], 1.0,
                         want_acc=True, want_out=False, groups=groups,
                         a_gstride=cgw.stride(0) * O, b_gstride=xp.stride(0) * I)
    reducer.sum_acc(acc)
    gw = dequant(acc, scales[2:3], scales[0:1], 1.0 / batch_global)
    # ---- dX: W is replicated, its scale is already global
    cw, kw, sw, _ = ops.quant_proj_rows(w if w.dtype == torch.float32 else w.float(), 1, O, I, 0xFFFF, bits_gx)
    gx, _ = ops.gemm_i8(cgx, cw, b * L, I, ops.pad16(O), bits_gx, bits_gx, scales[1:2], sw, 1.0, exact=True)
    return GradPair(gx.reshape(b, L, I), gw)


def self_group(reducer: Reducer):
    return reducer.group if reducer.group is not None else dist.group.WORLD
