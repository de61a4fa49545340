"""Drop-in torch modules whose backward is the HLQ path on B200.

Mirror of the reference's GEMM-layer hooks (harness/layers.py:22-93):
forward = stock ``F.linear`` plus ACBP compression of the input
(``GemmLayer._store_forward``, layers.py:46-55); backward = HLQ
(``GemmLayer._strategy_backward``, layers.py:57-69): the int8 low-rank weight
gradient from the compressed activation and the int4 Hadamard-quantized input
gradient, both on the sm_100a kernels.  The raw input is not kept.

Conventions:
  * 2-D input (N, I) is viewed as (N, 1, I) (layers.py:87) -> projection along N;
    >3-D input uses B = shape[0], L = prod(shape[1:-1]);
  * torch's mean-loss gradient already carries 1/B, so the dW dequant uses
    extra = 1 (the reference applies 1/B inside hlq_grad_weight, layers.py:239-250);
  * dX is produced in the input's dtype (bf16 under autocast) with the fp32
    epilogue; dW is fp32 (the master weight's dtype); the bias gradient is a
    plain torch reduction.
"""
from __future__ import annotations

import os

import torch
import torch.nn as nn
import torch.nn.functional as F

from . import ops
from .backprop import BackwardStrategy, dual_ok, ht_axis_for, _proj_view
from .errors import ParameterError


def _blv(shape):
    if len(shape) == 2:
        return shape[0], 1, shape[1]
    if len(shape) < 2:
        raise ParameterError(f"HLQ linear needs at least 2-D input, got {tuple(shape)}")
    L = 1
    for s in shape[1:-1]:
        L *= s
    return shape[0], L, shape[-1]


_SIDE = {}
PACK_GX = [None]  # None: HLQ_PACK_GX from the environment (default off); True / False: forced


def pack_gx_enabled() -> bool:
    """Whether the training path keeps the 4-bit gx codes packed two per byte."""
    if PACK_GX[0] is not None:
        return bool(PACK_GX[0])
    return os.environ.get("HLQ_PACK_GX", "0") == "1"
_STAGES = [None]  # list sink while capture_stages() is active


class capture_stages:
    """Record, per HLQLinearFunction.backward call, the codes and scales the
    training path computed (parity tests of the path that actually trains).
    The tensors are views, not copies; no extra kernels run."""

    def __enter__(self):
        self.records = []
        _STAGES[0] = self.records
        return self.records

    def __exit__(self, *exc):
        _STAGES[0] = None
        return False


def side_stream(device) -> torch.cuda.Stream:
    """Auxiliary stream for the forward ACBP / backward dW work when
    HLQ_SIDE_STREAM=1.  Default: the current stream.  The persistent GEMMs and
    the cooperative transform kernels each fill every SM, so a second stream
    buys no real overlap (0.4 ms/step at best on ViT-B/16), and with the host
    running several steps ahead the cross-stream interleaving made the step
    time erratic (40-86 ms/step, B200) -- one stream gives a steady 40.8 ms."""
    if os.environ.get("HLQ_SIDE_STREAM", "0") != "1":
        return torch.cuda.current_stream(device)
    key = torch.device(device).index
    if key not in _SIDE:
        _SIDE[key] = torch.cuda.Stream(device=device)
    return _SIDE[key]


class HLQLinearFunction(torch.autograd.Function):
    """y = x W^T + b forward; HLQ backward (ACBP payload saved, raw x dropped).

    Forward computes ACBP(X) and takes the W codes of the dX product (from the
    model-wide batched refresh, or a per-layer transform): codes taken at
    forward time are the codes of the W the backward differentiates (an
    in-place update in between trips autograd's version check on the saved
    weight)."""

    @staticmethod
    def forward(ctx, x, weight, bias, strategy: BackwardStrategy, wcodes=None, calib_layer=None, dp=None):
        B, L, I = _blv(x.shape)
        O = weight.shape[0]
        plan = strategy.plan
        bits_gw = strategy.grad_weight_path.bits or 8
        bits_gx = strategy.grad_input_path.bits or 4
        axis = ht_axis_for(B, L, plan.block_size, strategy.pad_small_axes)
        segs, rows, cols, ld_src, seg_src = _proj_view(B, L, I, axis)
        main = torch.cuda.current_stream()
        side = side_stream(x.device)
        side.wait_stream(main)
        payload = sx = cw = sw = None
        k = 0
        with torch.cuda.stream(side):
            if ctx.needs_input_grad[1] and dp is not None:
                # exact data-parallel mode: the scale of the WHOLE batch's projection (dp.ExactDP)
                if axis == 0 and B % plan.block_size:
                    raise ParameterError("exact DP with the batch-axis projection needs shards of a multiple "
                                         f"of {plan.block_size} samples, got {B}")
                payload, k, sx = dp.quant_rows(x.detach().contiguous(), segs, rows, cols, ld_src, seg_src,
                                               plan.gpu_bitmap(), bits_gw)
            elif ctx.needs_input_grad[1]:
                payload, k, sx, _ = ops.quant_proj_rows(x.detach().contiguous(), segs, rows, cols,
                                                        plan.gpu_bitmap(), bits_gw, ld_src, seg_src,
                                                        want_stats=False)
            if ctx.needs_input_grad[0] and wcodes is not None:
                cw, sw = wcodes[0], wcodes[1]  # refreshed for this weight version by refresh_weight_codes
            elif ctx.needs_input_grad[0]:
                w32 = weight.detach() if weight.dtype == torch.float32 else weight.detach().float()
                cw, _, sw, _ = ops.quant_proj_rows(w32, 1, O, I, 0xFFFF, bits_gx)
        if x.dtype == weight.dtype:
            wx = weight
        elif wcodes is not None and len(wcodes) > 2 and wcodes[2] is not None and x.dtype == torch.bfloat16:
            wx = wcodes[2]  # bf16 copy written by the batched codes refresh (no per-layer cast)
        else:
            wx = weight.to(x.dtype)
        y = F.linear(x, wx, None if bias is None else bias.to(x.dtype))
        main.wait_stream(side)
        for t in (payload, sx, cw, sw):
            if t is not None:
                t.record_stream(main)
        x.record_stream(side)
        ctx.save_for_backward(weight, payload, sx, cw, sw)
        ctx.meta = (B, L, I, axis, k, x.dtype, tuple(x.shape), bias is not None, strategy)
        ctx.calib_layer = calib_layer
        ctx.dp = dp
        return y

    @staticmethod
    def backward(ctx, gy):
        weight, payload, sx, cw_saved, sw_saved = ctx.saved_tensors
        B, L, I, axis, k, x_dtype, x_shape, has_bias, strategy = ctx.meta
        O = weight.shape[0]
        gy3 = gy.reshape(B, L, O)
        if gy3.dtype not in (torch.float32, torch.bfloat16):
            gy3 = gy3.float()
        gy3 = gy3.contiguous()
        if ctx.calib_layer is not None:  # calibrate_bases: the layer's gradient-energy hook (layers.py:61-62)
            _calib_record(ctx.calib_layer, gy3, axis)
        gx = gw = gb = None
        bits_gx = strategy.grad_input_path.bits or 4
        bits_gw = strategy.grad_weight_path.bits or 8
        out_dtype = x_dtype if x_dtype in (torch.float32, torch.bfloat16) else torch.float32
        if ctx.dp is not None and ctx.needs_input_grad[1]:
            return _exact_dp_backward(ctx, gy, gy3, weight, payload, sx, cw_saved, sw_saved)
        if ctx.needs_input_grad[0] and ctx.needs_input_grad[1] and dual_ok(B, L, axis):
            # one fused transform of gy feeds both products (2 reads of gy instead of 4)
            segs, rows, cols, ld_src, seg_src = _proj_view(B, L, O, axis)
            want_gb = has_bias and ctx.needs_input_grad[2]
            # 4-bit gx codes packed two per byte in HBM (the dX GEMM widens them in smem):
            # half the code bytes, bit-identical results, but measured 12-15 % slower dX GEMMs
            # and a ~1 % slower ViT-B/16 step on B200 -- opt-in (PACK_GX / HLQ_PACK_GX=1)
            pack = bits_gx == 4 and pack_gx_enabled()
            # the bias gradient (column sums of gy) comes out of the same kernel's STATS pass
            cgx, sgx, cg, kg, sg, _, *cs = ops.quant_dual(gy3, segs, rows, cols,
                                                          strategy.plan.gpu_bitmap(), bits_gx, bits_gw,
                                                          ld_src, seg_src, colsum=want_gb, pack_gx=pack,
                                                          want_stats=False)
            cw, sw = cw_saved, sw_saved
            # the two products are independent: dW on the side stream, dX here
            main = torch.cuda.current_stream()
            side = side_stream(gy.device)
            side.wait_stream(main)
            # (torch.cuda.current_stream() returns a fresh wrapper per call: compare handles)
            if side.cuda_stream == main.cuda_stream and ops.pair_eligible(O, B * L, k, ops.pad16(O), I, I):
                # dW and dX as one CTA-pair launch over both products' tiles when each
                # contraction is long or its output wide (ops.pair_eligible; otherwise two
                # gemm_i8 calls, which keep the split-K planner)
                gw, gx = ops.gemm_i8_pair(
                    dict(a=cg, b=payload, m=O, n=I, k=k, bits_a=bits_gw, bits_b=bits_gw, sa=sg, sb=sx),
                    dict(a=cgx, b=cw, m=B * L, n=I, k=ops.pad16(O), bits_a=bits_gx, bits_b=bits_gx, sa=sgx,
                         sb=sw, out_dtype=out_dtype, a_packed=pack))
            else:
                with torch.cuda.stream(side):
                    gw, _ = ops.gemm_i8(cg, payload, O, I, k, bits_gw, bits_gw, sg, sx, 1.0, exact=False)
                gx, _ = ops.gemm_i8(cgx, cw, B * L, I, ops.pad16(O), bits_gx, bits_gx, sgx, sw, 1.0,
                                    exact=False, out_dtype=out_dtype, a_packed=pack)
            main.wait_stream(side)
            gw.record_stream(main)
            for t in (cg, sg, payload, sx):
                t.record_stream(side)
            if _STAGES[0] is not None:
                # parity capture of the training path, in the reference's layouts
                # (backprop.py:350-410: codes (T, O_p), (O_p, I), (O, K), payload (K, I))
                _STAGES[0].append(dict(gx_codes_g=ops.unpack_int4(cgx, ops.pad16(O)) if pack else cgx[:, :ops.pad16(O)],
                                       gx_scale_g=sgx, gx_packed=pack,
                                       gx_codes_w=cw[:, :ops.pad16(O)].t(), gx_scale_w=sw,
                                       gw_codes_g=cg[:, :k], gw_scale_g=sg, x_codes=payload[:, :k].t(),
                                       x_scale=sx, axis=axis))
            if weight.dtype != torch.float32:
                gw = gw.to(weight.dtype)
            gx = gx.reshape(x_shape).to(x_dtype)
            if want_gb:
                gb = cs[0]
            return gx, gw, gb, None, None, None, None
        if ctx.needs_input_grad[1]:
            bits = strategy.grad_weight_path.bits or 8
            segs, rows, cols, ld_src, seg_src = _proj_view(B, L, O, axis)
            cg, kg, sg, _ = ops.quant_proj_rows(gy3, segs, rows, cols, strategy.plan.gpu_bitmap(),
                                                bits, ld_src, seg_src)
            groups = L if axis == 0 else 1
            gw, _ = ops.gemm_i8(cg, payload, O, I, k, bits, bits, sg, sx, 1.0, exact=False,
                                out_dtype=torch.float32, groups=groups,
                                a_gstride=cg.stride(0) * O, b_gstride=payload.stride(0) * I)
            if weight.dtype != torch.float32:
                gw = gw.to(weight.dtype)
        if ctx.needs_input_grad[0]:
            bits = strategy.grad_input_path.bits or 4
            cgx, sgx, _ = ops.quant_ht_cols(gy3.reshape(B * L, O), bits)
            cw, sw = cw_saved, sw_saved
            out_dtype = x_dtype if x_dtype in (torch.float32, torch.bfloat16) else torch.float32
            gx, _ = ops.gemm_i8(cgx, cw, B * L, I, ops.pad16(O), bits, bits, sgx, sw, 1.0,
                                exact=False, out_dtype=out_dtype)
            gx = gx.reshape(x_shape)
            if gx.dtype != x_dtype:
                gx = gx.to(x_dtype)
        if has_bias and ctx.needs_input_grad[2]:
            gb = gy.reshape(-1, O).sum(0, dtype=torch.float32)
        return gx, gw, gb, None, None, None, None


def _exact_dp_backward(ctx, gy, gy3, weight, payload, sx, cw, sw):
    """HLQLinearFunction.backward in the exact data-parallel mode (dp.ExactDP):
    global-scale gy codes, dW = all-reduce(SUM) of the int32 accumulators
    (asynchronous, overlapped with the local dX GEMM) + one dequant."""
    B, L, I, axis, k, x_dtype, x_shape, has_bias, strategy = ctx.meta
    dp = ctx.dp
    O = weight.shape[0]
    bits_gx = strategy.grad_input_path.bits or 4
    bits_gw = strategy.grad_weight_path.bits or 8
    cgx, sgx, cg, kg, sg = dp.quant_gy(gy3, axis, strategy.plan.gpu_bitmap(), bits_gx, bits_gw)
    groups = L if axis == 0 else 1
    _, acc = ops.gemm_i8(cg, payload, O, I, k, bits_gw, bits_gw, sg, sx, 1.0, want_acc=True, want_out=False,
                         groups=groups, a_gstride=cg.stride(0) * O, b_gstride=payload.stride(0) * I)
    acc, work = dp.reduce_acc_async(acc, k, groups, bits_gw)
    gx = None
    if ctx.needs_input_grad[0]:
        out_dtype = x_dtype if x_dtype in (torch.float32, torch.bfloat16) else torch.float32
        gx, _ = ops.gemm_i8(cgx, cw, B * L, I, ops.pad16(O), bits_gx, bits_gx, sgx, sw, 1.0, exact=False,
                            out_dtype=out_dtype)
        gx = gx.reshape(x_shape).to(x_dtype)
    work.wait()
    gw = dp.dequant_fast(acc, sg, sx, weight.dtype)
    gb = gy.reshape(-1, O).sum(0, dtype=torch.float32) if has_bias and ctx.needs_input_grad[2] else None
    return gx, gw, gb, None, None, None, None


class BaselineLinearFunction(torch.autograd.Function):
    """Linear layer under a baseline strategy (naive quant, HQ, LBP-WHT, float
    pipelines; backprop.py:91-155): the raw input is saved and the backward is
    backprop.strategy_backward on the hlq_xform / GEMM kernels -- the
    reference's ablation-grid path (harness/layers.py:57-69 with
    store_compressed off)."""

    @staticmethod
    def forward(ctx, x, weight, bias, strategy: BackwardStrategy, rng=None):
        ctx.save_for_backward(x, weight)
        ctx.meta = (tuple(x.shape), bias is not None, strategy, rng)
        return F.linear(x, weight.to(x.dtype) if x.dtype != weight.dtype else weight,
                        None if bias is None else bias.to(x.dtype))

    @staticmethod
    def backward(ctx, gy):
        from .backprop import strategy_backward
        x, weight = ctx.saved_tensors
        x_shape, has_bias, strategy, rng = ctx.meta
        B, L, I = _blv(x_shape)
        O = weight.shape[0]
        gp = strategy_backward(x.reshape(B, L, I).float(), weight.float(), gy.reshape(B, L, O).float(), strategy,
                               rng=rng, gw_scale=1.0)
        gb = gy.reshape(-1, O).sum(0, dtype=torch.float32) if has_bias and ctx.needs_input_grad[2] else None
        return gp.grad_input.reshape(x_shape).to(x.dtype), gp.grad_weight.to(weight.dtype), gb, None, None


class HLQLinear(nn.Linear):
    """nn.Linear with the HLQ backward (reference harness/layers.py:72-93)."""

    def __init__(self, in_features: int, out_features: int, bias: bool = True,
                 strategy: BackwardStrategy | None = None, device=None, dtype=None):
        super().__init__(in_features, out_features, bias=bias, device=device, dtype=dtype)
        self.strategy = strategy or BackwardStrategy.hlq()
        self._wcodes = None  # (weight version, data_ptr, bits, codes, scale)
        self._hlq_weight_codes = True  # refreshed in batch by refresh_weight_codes
        self.dp = None  # dp.ExactDP when the exact data-parallel mode is on (dp.enable_exact_dp)

    def bits_gx(self) -> int:
        return self.strategy.grad_input_path.bits or 4

    def cached_weight_codes(self):
        """(codes, scale) of the current weight if refresh_weight_codes made
        them for this exact weight version, else None."""
        c = self._wcodes
        w = self.weight
        if c is not None and c[0] == w._version and c[1] == w.data_ptr() and c[2] == self.bits_gx():
            return c[3:]
        return None

    def forward(self, x):
        if not (self.training and torch.is_grad_enabled()):
            return F.linear(x, self.weight.to(x.dtype), None if self.bias is None else self.bias.to(x.dtype))
        if torch.is_autocast_enabled("cuda"):
            x = x.to(torch.get_autocast_dtype("cuda"))
        with torch.autocast("cuda", enabled=False):
            if not self.strategy.is_hlq:
                return BaselineLinearFunction.apply(x, self.weight, self.bias, self.strategy)
            return HLQLinearFunction.apply(x, self.weight, self.bias, self.strategy, self.cached_weight_codes(),
                                           self if _CALIB[0] is not None else None, self.dp)

    @classmethod
    def from_linear(cls, lin: nn.Linear, strategy: BackwardStrategy | None = None) -> "HLQLinear":
        m = cls(lin.in_features, lin.out_features, bias=lin.bias is not None, strategy=strategy,
                device=lin.weight.device, dtype=lin.weight.dtype)
        with torch.no_grad():
            m.weight.copy_(lin.weight)
            if lin.bias is not None:
                m.bias.copy_(lin.bias)
        return m


_CALIB = [None]  # {HLQLinear: [energy sums (16,) fp64, count]} while calibrate_bases runs


def calibrate_bases(model: nn.Module, backward_pass) -> dict:
    """One-batch L1 basis selection (harness/train.py:137-167): run
    ``backward_pass()`` (a forward + backward of one calibration batch) while
    every HLQLinear records the per-basis |coefficient| energy of its upstream
    gradient along its projection axis (GPU, hlq_basis_energy), then give each
    layer the `rank` bases carrying the most energy (select_bases).  Returns
    {layer: basis tuple}; full-rank plans are left alone."""
    from .hadamard import select_bases
    layers = [m for m in model.modules() if isinstance(m, HLQLinear)]
    _CALIB[0] = {m: None for m in layers}
    try:
        backward_pass()
    finally:
        sinks, _CALIB[0] = _CALIB[0], None
    out = {}
    for m in layers:
        plan = m.strategy.plan
        if plan.full_rank or sinks.get(m) is None:
            continue
        sums, count = sinks[m]
        idx = select_bases((sums / max(count, 1)).cpu().numpy(), plan.rank)
        m.strategy = m.strategy.with_plan(plan.with_bases(idx))
        out[m] = idx
    return out


def _calib_record(layer, gy3, axis: int):
    sinks = _CALIB[0]
    if sinks is None or layer not in sinks:
        return
    B, L, O = gy3.shape
    segs, rows, cols, ld_src, seg_src = _proj_view(B, L, O, axis)
    e, n = ops.basis_energy(gy3, segs, rows, cols, ld_src, seg_src)
    prev = sinks[layer]
    sinks[layer] = (e, n) if prev is None else (prev[0] + e, prev[1] + n)


def refresh_weight_codes(module: nn.Module, force: bool = False) -> int:
    """Recompute, in ONE batched launch per bit width (hlq_quantize_weights),
    the dX weight codes Q(HT_O(W)) of every HLQLinear under `module` whose
    weight changed since its codes were made (training: every layer, once per
    optimizer step).  HLQLinear.forward then reuses them instead of launching
    a per-layer transform.  Returns the number of layers refreshed."""
    stale = {}
    # under CUDA-graph capture the refresh must be part of the captured step whatever
    # the cache says (replays re-run the kernels, not this Python check)
    force = force or (torch.cuda.is_available() and torch.cuda.is_current_stream_capturing())
    for m in module.modules():
        # HLQLinear and HLQConv2d (its weight viewed as (O, C*k*k), the dX operand's layout)
        if getattr(m, "_hlq_weight_codes", False) and m.weight.is_cuda and \
                (force or m.cached_weight_codes() is None):
            stale.setdefault(m.bits_gx(), []).append(m)
    n = 0
    for bits, mods in stale.items():
        ws = [(m.weight.detach() if m.weight.dtype == torch.float32 else m.weight.detach().float())
              .reshape(m.weight.shape[0], -1) for m in mods]
        # Linear layers under autocast also take the bf16 weight for their forward GEMM
        want_bf16 = torch.is_autocast_enabled("cuda") and torch.get_autocast_dtype("cuda") == torch.bfloat16 \
            and os.environ.get("HLQ_WCODES_BF16", "1") != "0"
        for m, res in zip(mods, ops.quant_weights(ws, bits, bf16=want_bf16)):
            wbf = res[2] if want_bf16 and isinstance(m, HLQLinear) else None
            m._wcodes = (m.weight._version, m.weight.data_ptr(), bits, res[0], res[1], wbf)
        n += len(mods)
    return n


def _refresh_hook(module, args):
    # always recompute: the (version, data_ptr) key cannot see in-place writes through
    # `.data` (EMA, custom optimizers, storage swaps), and in training every step
    # changes every weight anyway, so the cache would only skip work for extra
    # forwards within one step
    if module.training and torch.is_grad_enabled():
        refresh_weight_codes(module, force=True)


def convert_linears(module: nn.Module, strategy: BackwardStrategy | None = None,
                    batch_weight_codes: bool = True) -> nn.Module:
    """Swap every nn.Linear under `module` for HLQLinear (in place).  With
    batch_weight_codes, `module` also gets a forward pre-hook that refreshes
    all its layers' weight codes in one launch per training forward
    (refresh_weight_codes)."""
    _convert(module, strategy)
    if batch_weight_codes and not getattr(module, "_hlq_wcodes_hook", False):
        module.register_forward_pre_hook(_refresh_hook)
        module._hlq_wcodes_hook = True
    return module


def _convert(module: nn.Module, strategy):
    for name, child in list(module.named_children()):
        if isinstance(child, nn.Linear) and not isinstance(child, HLQLinear):
            setattr(module, name, HLQLinear.from_linear(child, strategy))
        else:
            _convert(child, strategy)
