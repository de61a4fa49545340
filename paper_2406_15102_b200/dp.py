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
