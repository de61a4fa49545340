"""Conv2d on the HLQ path (reference harness/layers.py:96-158).

The reference lowers Conv2d to its Linear path: cols = im2col(x) (B, L=Ho*Wo,
I=C*k*k, column c*k*k + i*k + j), ACBP on cols at forward time, and at backward
gy (B, O, Ho, Wo) -> (B, L, O), strategy_backward, col2im.  Here:

  forward   y = F.conv2d(x, w) (cuDNN) + ACBP of im2col(x) straight from
            channels-last x (hlq_conv_acbp_compress, no cols tensor);
  backward  one fused transform of gy (channels-last = (B, L, O) contiguous):
            gx codes Q4(HT_O) and gw codes Q8(P_L); W codes Q4(HT_O(W));
            dW = int8 GEMM(gw codes, payload) -> (O, C, k, k);
            dcols = int8 GEMM(gx codes, W codes); dX = col2im(dcols) in the
            reference's tap order (bit-exact for fp32 dcols).

Square kernels, integer stride / padding, no dilation or groups -- the
reference's Conv2d surface (layers.py:124-139).
"""
from __future__ import annotations

import torch
import torch.nn as nn
import torch.nn.functional as F

from . import ops
from .backprop import ACBPActivation, BackwardStrategy, QuantizedTensor, ht_axis_for, _proj_view
from .errors import DimensionError, ParameterError


def _to_nhwc(x: torch.Tensor) -> torch.Tensor:
    """(B, H, W, C) contiguous view of x (free when x is channels_last)."""
    return x.permute(0, 2, 3, 1).contiguous()


def conv_acbp_compress(x: torch.Tensor, k: int, stride: int, pad: int, strategy: BackwardStrategy, dp=None,
                       want_stats: bool = True):
    """ACBP of im2col(x) (layers.py:141-151 + backprop.py:373-385).  Returns an
    ACBPActivation whose orig_shape is the lowered (B, L, C*k*k).  dp
    (dp.ExactDP): the scale of the whole data-parallel batch (amax is then None)."""
    B, C, H, W = x.shape
    Ho, Wo = ops.conv_out_hw(H, W, k, stride, pad)
    L = Ho * Wo
    plan = strategy.plan
    bits = strategy.grad_weight_path.bits or 8
    axis = ht_axis_for(B, L, plan.block_size, strategy.pad_small_axes)
    if axis == 1 and C * k * k <= 256 and (C * x.element_size()) % 16 != 0:
        # few input channels (e.g. an RGB stem): materialise the small cols tensor and run
        # the TMA projection on it -- the im2col producer's 256-channel tiles would be
        # almost empty and the gather fallback handles 16-byte-unaligned pixels slowly
        I = C * k * k
        ldc = (I + 7) // 8 * 8
        Ho, Wo = ops.conv_out_hw(H, W, k, stride, pad)
        xp = F.pad(x, (pad, pad, pad, pad))
        sb, sc, sh, sw = xp.stride()
        # cols[b, (ho, wo), (c, i, j)] = xp[b, c, ho*s + i, wo*s + j] -- one strided copy
        # (F.unfold runs one kernel per image)
        win = xp.as_strided((B, Ho, Wo, C, k, k), (sb, stride * sh, stride * sw, sc, sh, sw))
        cols = torch.zeros((B, L, ldc), dtype=x.dtype, device=x.device)
        cols[:, :, :I] = win.reshape(B, L, I)
        if dp is not None:
            codes, kk, scale = dp.quant_rows(cols, B, L, I, ldc, L * ldc, plan.gpu_bitmap(), bits)
            amax = None
        else:
            codes, kk, scale, amax = ops.quant_proj_rows(cols, B, L, I, plan.gpu_bitmap(), bits, ldc, L * ldc)
    elif axis == 1 and dp is not None:
        codes, kk, scale = dp.quant_conv(_to_nhwc(x), k, stride, pad, plan.gpu_bitmap(), bits)
        amax = None
    elif axis == 1:
        codes, kk, scale, amax = ops.conv_acbp(_to_nhwc(x), k, stride, pad, plan.gpu_bitmap(), bits,
                                               want_stats=want_stats)
    else:
        # L < 16: projection along the batch axis needs the lowered tensor itself
        cols = F.unfold(x, k, padding=pad, stride=stride).transpose(1, 2).contiguous()
        segs, rows, cols_, ld, sg = _proj_view(B, L, C * k * k, axis)
        if dp is not None:
            if B % plan.block_size:
                raise ParameterError("exact DP with the batch-axis projection needs shards of a multiple "
                                     f"of {plan.block_size} images, got {B}")
            codes, kk, scale = dp.quant_rows(cols, segs, rows, cols_, ld, sg, plan.gpu_bitmap(), bits)
            amax = None
        else:
            codes, kk, scale, amax = ops.quant_proj_rows(cols, segs, rows, cols_, plan.gpu_bitmap(), bits,
                                                         ld, sg)
    q = QuantizedTensor(payload=codes, bits=bits, scale=scale)
    return ACBPActivation(quantized=q, orig_shape=(B, L, C * k * k), axis=axis, plan=plan, k=kk), amax


def _conv_backward(acbp: ACBPActivation, w4: torch.Tensor, gy: torch.Tensor, x_shape, stride: int,
                   pad: int, strategy: BackwardStrategy, extra: float, exact: bool, dx_dtype,
                   need_dx: bool = True, need_dw: bool = True, stages: dict | None = None,
                   implicit: bool | None = None, wcodes=None, dp=None):
    """implicit (default: not exact): dX as implicit GEMMs over the taps
    (hlq_conv_dgrad_i8_ex -- one launch, or stride^2 output phases; taps summed
    in int32, matches the reference to fp32 rounding); otherwise the
    reference's lowering, GEMM -> dcols -> col2im in tap order (bit-exact with
    the exact epilogue)."""
    B, C, H, W = x_shape
    O, _, k, _ = w4.shape
    Ho, Wo = gy.shape[2], gy.shape[3]
    L = Ho * Wo
    I = C * k * k
    bits_gx = strategy.grad_input_path.bits or 4
    bits_gw = strategy.grad_weight_path.bits or 8
    gy3 = _to_nhwc(gy)
    if gy3.dtype not in (torch.float32, torch.bfloat16):
        gy3 = gy3.float()
    segs, rows, cols, ld_src, seg_src = _proj_view(B, L, O, acbp.axis)
    dx = dw = None
    want = stages is not None
    if dp is not None:
        # exact data-parallel mode: both gy operands with the whole batch's scales
        cgx, sgx, cg, kg, sg = dp.quant_gy(gy3.reshape(B, L, O), acbp.axis, acbp.plan.gpu_bitmap(), bits_gx,
                                           bits_gw)
    elif acbp.axis == 1:
        cgx, sgx, cg, kg, sg, _ = ops.quant_dual(gy3, segs, rows, cols, acbp.plan.gpu_bitmap(),
                                                 bits_gx, bits_gw, ld_src, seg_src, want_stats=False)
    else:
        cg, kg, sg, _ = ops.quant_proj_rows(gy3, segs, rows, cols, acbp.plan.gpu_bitmap(), bits_gw,
                                            ld_src, seg_src)
        cgx, sgx, _ = ops.quant_ht_cols(gy3.reshape(B * L, O), bits_gx)
    if kg != acbp.k:
        raise DimensionError("projected extents differ between forward and backward")
    pending = None
    if need_dw:
        groups = L if acbp.axis == 0 else 1
        xp = acbp.quantized.payload
        if dp is not None:
            # exact int32 partial sums, all-reduced under the dX GEMM, one dequant
            _, accw = ops.gemm_i8(cg, xp, O, I, kg, bits_gw, bits_gw, sg, acbp.quantized.scale, 1.0,
                                  want_acc=True, want_out=False, groups=groups,
                                  a_gstride=cg.stride(0) * O, b_gstride=xp.stride(0) * I)
            pending = dp.reduce_acc_async(accw, kg, groups, bits_gw)
        else:
            dw2, accw = ops.gemm_i8(cg, xp, O, I, kg, bits_gw, bits_gw, sg, acbp.quantized.scale, extra,
                                    exact=exact, want_acc=want, groups=groups,
                                    a_gstride=cg.stride(0) * O, b_gstride=xp.stride(0) * I)
            dw = dw2.reshape(O, C, k, k)
            if want:
                stages.update(gw_codes_g=cg[:, :kg], gw_scale_g=sg, gw_acc=accw)
    if implicit is None:
        implicit = not exact and pad <= k - 1
    if need_dx and (wcodes is not None and not want):
        cw, sw = wcodes  # batched refresh (layers.refresh_weight_codes) for this weight version
        kw = O
    elif need_dx:
        w2 = w4.detach().reshape(O, I)
        w2 = w2 if w2.dtype == torch.float32 else w2.float()
        cw, kw, sw, _ = ops.quant_proj_rows(w2.contiguous(), 1, O, I, 0xFFFF, bits_gx)
    if need_dx and implicit:
        dx_nhwc, accx = ops.conv_dgrad_i8(cgx, B, Ho, Wo, O, cw, C, k, pad, bits_gx, sgx, sw, exact=exact,
                                          out_dtype=dx_dtype, want_acc=want, stride=stride, H=H, W=W)
        dx = dx_nhwc.permute(0, 3, 1, 2)  # NCHW shape, channels_last memory
        if want:
            stages.update(gx_codes_g=cgx, gx_scale_g=sgx, gx_codes_w=cw[:, :kw].t(), gx_scale_w=sw,
                          dx_acc=accx)
    elif need_dx:
        # fp32 dcols even for training: rounding every tap's partial to bf16 before the
        # col2im sum costs ~1.6e-3 relative error on dX, over the 1e-3 contract
        cols_dtype = torch.float32
        # training path: W codes rows tap-major, so dcols columns are (tap, c) and the
        # col2im reads each tap's channels contiguously (same per-element sum order);
        # the reference-mirroring path keeps the reference's (c, tap) column order
        tap_major = not want and C % 8 == 0
        cwg = cw.view(C, k * k, cw.shape[1]).transpose(0, 1).reshape(I, cw.shape[1]) if tap_major else cw
        dcols, accx = ops.gemm_i8(cgx, cwg, B * L, I, ops.pad16(O), bits_gx, bits_gx, sgx, sw, 1.0,
                                  exact=exact, out_dtype=cols_dtype, want_acc=want)
        dx_nhwc = ops.col2im(dcols, B, H, W, C, k, stride, pad, out_dtype=dx_dtype, tap_major=tap_major)
        dx = dx_nhwc.permute(0, 3, 1, 2)  # NCHW shape, channels_last memory
        if want:
            stages.update(gx_codes_g=cgx, gx_scale_g=sgx, gx_codes_w=cw[:, :kw].t(), gx_scale_w=sw,
                          gx_acc=accx, dcols=dcols)
    if pending is not None:
        acc, work = pending
        work.wait()
        dw = dp.dequant_fast(acc, sg, acbp.quantized.scale).reshape(O, C, k, k)
    return dx, dw


def conv2d_hlq_backward(x: torch.Tensor, w4: torch.Tensor, gy: torch.Tensor, stride: int, pad: int,
                        strategy: BackwardStrategy | None = None, stages: dict | None = None):
    """Reference Conv2d forward(ACBP) + backward (layers.py:141-158) on the GPU,
    reference conventions (1/B on dW, fp32, exact epilogue): returns (dX (B,C,H,W), dW (O,C,k,k))."""
    strategy = strategy or BackwardStrategy.hlq()
    if x.dim() != 4 or w4.dim() != 4 or gy.dim() != 4 or w4.shape[2] != w4.shape[3]:
        raise DimensionError("expected x (B,C,H,W), square w (O,C,k,k), gy (B,O,Ho,Wo)")
    B, C, H, W = x.shape
    O, Cw, k, _ = w4.shape
    if Cw != C:
        raise DimensionError(f"weight {tuple(w4.shape)} does not match {C} input channels")
    Ho, Wo = ops.conv_out_hw(H, W, k, stride, pad)
    if tuple(gy.shape) != (B, O, Ho, Wo):
        raise DimensionError(f"gy {tuple(gy.shape)} does not match ({B}, {O}, {Ho}, {Wo})")
    acbp, amax = conv_acbp_compress(x, k, stride, pad, strategy)
    ops.check_finite(amax)
    if stages is not None:
        stages.update(x_codes=acbp.reference_payload(), x_scale=acbp.quantized.scale, axis=acbp.axis)
    return _conv_backward(acbp, w4, gy, x.shape, stride, pad, strategy, 1.0 / B, True, torch.float32,
                          stages=stages)


class HLQConv2dFunction(torch.autograd.Function):
    @staticmethod
    def forward(ctx, x, weight, bias, stride, pad, strategy: BackwardStrategy, wcodes=None, dp=None):
        y = F.conv2d(x, weight.to(x.dtype), None if bias is None else bias.to(x.dtype),
                     stride=stride, padding=pad)
        ctx.wcodes = wcodes if ctx.needs_input_grad[0] else None
        acbp = None
        if ctx.needs_input_grad[1]:
            acbp, _ = conv_acbp_compress(x.detach(), weight.shape[2], stride, pad, strategy, dp=dp,
                                         want_stats=False)
            ctx.save_for_backward(weight, acbp.quantized.payload, acbp.quantized.scale)
        else:
            ctx.save_for_backward(weight, None, None)
        ctx.meta = (tuple(x.shape), x.dtype, stride, pad, strategy, bias is not None,
                    None if acbp is None else (acbp.axis, acbp.k, acbp.orig_shape))
        ctx.dp = dp
        return y

    @staticmethod
    def backward(ctx, gy):
        weight, payload, sx = ctx.saved_tensors
        x_shape, x_dtype, stride, pad, strategy, has_bias, am = ctx.meta
        dx = dw = db = None
        if am is None:
            # no weight gradient requested: dX only (dense path is the stock op)
            dx = torch.nn.grad.conv2d_input(x_shape, weight.to(gy.dtype), gy, stride=stride,
                                            padding=pad)
            return dx, None, None, None, None, None, None, None
        axis, kk, orig = am
        acbp = ACBPActivation(QuantizedTensor(payload, strategy.grad_weight_path.bits or 8, sx), orig,
                              axis, strategy.plan, kk)
        out_dtype = x_dtype if x_dtype in (torch.float32, torch.bfloat16) else torch.float32
        dx, dw = _conv_backward(acbp, weight, gy, x_shape, stride, pad, strategy, 1.0, False,
                                out_dtype, need_dx=ctx.needs_input_grad[0], wcodes=ctx.wcodes, dp=ctx.dp)
        if dx is not None and dx.dtype != x_dtype:
            dx = dx.to(x_dtype)
        if weight.dtype != torch.float32:
            dw = dw.to(weight.dtype)
        if has_bias and ctx.needs_input_grad[2]:
            db = gy.sum(dim=(0, 2, 3), dtype=torch.float32)
        return dx, dw, db, None, None, None, None, None


class HLQConv2d(nn.Conv2d):
    """nn.Conv2d (square kernel, int stride/padding, no dilation/groups) with
    the HLQ backward; keep activations channels_last for copy-free lowering."""

    def __init__(self, *args, strategy: BackwardStrategy | None = None, **kw):
        super().__init__(*args, **kw)
        if self.groups != 1 or self.dilation != (1, 1) or self.kernel_size[0] != self.kernel_size[1] \
                or self.stride[0] != self.stride[1] or self.padding[0] != self.padding[1] \
                or isinstance(self.padding, str) or self.padding_mode != "zeros":
            raise ParameterError("HLQConv2d supports square kernels, equal int stride/padding, "
                                 "no dilation / groups (the reference Conv2d surface)")
        self.strategy = strategy or BackwardStrategy.hlq()
        self._wcodes = None  # (weight version, data_ptr, bits, codes, scale); see refresh_weight_codes
        self._hlq_weight_codes = True
        self.dp = None  # dp.ExactDP when the exact data-parallel mode is on (dp.enable_exact_dp)

    def bits_gx(self) -> int:
        return self.strategy.grad_input_path.bits or 4

    def cached_weight_codes(self):
        c = self._wcodes
        w = self.weight
        if c is not None and c[0] == w._version and c[1] == w.data_ptr() and c[2] == self.bits_gx():
            return c[3], c[4]
        return None

    def forward(self, x):
        if not (self.training and torch.is_grad_enabled()):
            return super().forward(x)
        if torch.is_autocast_enabled("cuda"):
            x = x.to(torch.get_autocast_dtype("cuda"))
        with torch.autocast("cuda", enabled=False):
            return HLQConv2dFunction.apply(x, self.weight, self.bias, self.stride[0], self.padding[0],
                                           self.strategy, self.cached_weight_codes(), self.dp)

    @classmethod
    def from_conv(cls, conv: nn.Conv2d, strategy: BackwardStrategy | None = None) -> "HLQConv2d":
        m = cls(conv.in_channels, conv.out_channels, conv.kernel_size, stride=conv.stride,
                padding=conv.padding, bias=conv.bias is not None, strategy=strategy,
                device=conv.weight.device, dtype=conv.weight.dtype)
        with torch.no_grad():
            m.weight.copy_(conv.weight)
            if conv.bias is not None:
                m.bias.copy_(conv.bias)
        return m


def convert_convs(module: nn.Module, strategy: BackwardStrategy | None = None) -> nn.Module:
    """Swap every eligible nn.Conv2d under `module` for HLQConv2d (in place)."""
    for name, child in list(module.named_children()):
        if isinstance(child, nn.Conv2d) and not isinstance(child, HLQConv2d):
            ok = (child.groups == 1 and child.dilation == (1, 1)
                  and child.kernel_size[0] == child.kernel_size[1]
                  and child.stride[0] == child.stride[1] and child.padding[0] == child.padding[1]
                  and not isinstance(child.padding, str))
            if ok:
                setattr(module, name, HLQConv2d.from_conv(child, strategy))
        else:
            convert_convs(child, strategy)
    return module
