"""HLQ backward for linear (or im2col'd convolution) layers on B200.

Same public surface as the reference module
/root/reference/pkg/src/hlq/backprop.py (names, argument meaning, error
classes), over torch CUDA tensors:

    acbp_compress(x, plan, bits=8, rng=None, pad_small_axes=False) -> ACBPActivation
    hq_grad_input(gy, w, bits, rng=None, block=16) -> Tensor (B, L, I)
    hlq_grad_weight(acbp, gy, bits=8, rng=None) -> Tensor (O, I)
    strategy_backward(x_or_acbp, w, gy, strategy, rng=None) -> GradPair
    hlq_backward(x_or_acbp, w, gy, strategy=None, rng=None) -> GradPair

Every quantized stage runs in libhlq_b200.so (sm_100a): block-Hadamard /
projection + amax + pseudo-stochastic quantizer kernels and the tcgen05
int8 GEMM with the fused dequant epilogue.  Outputs are fp32 and, with the
exact epilogue used here, bit-identical to the reference on the same inputs.

Differences from the reference, by design:
  * ``rng`` (true stochastic rounding, quantize.py:114-125) runs on the GPU
    (hlq_quantize_stochastic: numpy's Philox4x64-10 stream reproduced in CUDA),
    bit-identical to the reference's RngState draws; the fused dual transform
    of the pseudo mode is not used then (each operand has its own stream).
  * the ACBP payload is stored K-major ((I, K) instead of (K, I)), which is
    the tcgen05 operand layout; ``ACBPActivation.reference_payload()``
    returns the reference layout.
"""
from __future__ import annotations

from dataclasses import dataclass, field, replace

import torch

from . import ops
from .rng import TAG_GW_LEFT, TAG_GW_RIGHT, TAG_GX_LEFT, TAG_GX_RIGHT, site_key
from .errors import DimensionError, ParameterError, StateError
from .hadamard import DEFAULT_BLOCK, DEFAULT_RANK, HadamardPlan, lowest_sequency_bases

GX_MODES = ("fp", "quant", "ht_quant", "lowrank")
GW_MODES = ("fp", "quant", "ht_quant", "lowrank", "lowrank_quant")


@dataclass(frozen=True)
class GradPair:
    grad_input: torch.Tensor
    grad_weight: torch.Tensor


@dataclass(frozen=True)
class PathSpec:
    mode: str
    bits: int | None = None


@dataclass(frozen=True)
class BackwardStrategy:
    """Per-layer backward configuration (backprop.py:66-155)."""

    name: str
    grad_input_path: PathSpec
    grad_weight_path: PathSpec
    plan: HadamardPlan = field(default_factory=HadamardPlan)
    pad_small_axes: bool = False
    store_compressed: bool = True

    def __post_init__(self):
        gx, gw = self.grad_input_path, self.grad_weight_path
        if gx.mode not in GX_MODES:
            raise ParameterError(f"unknown grad_input mode {gx.mode!r}")
        if gw.mode not in GW_MODES:
            raise ParameterError(f"unknown grad_weight mode {gw.mode!r}")
        for spec in (gx, gw):
            if spec.mode in ("fp", "lowrank") and spec.bits is not None:
                raise ParameterError(f"mode {spec.mode!r} does not quantize; bits must be None")
            if spec.bits is not None and spec.bits not in (4, 8):
                raise ParameterError(f"bits must be 4 or 8, got {spec.bits}")

    @classmethod
    def vanilla(cls) -> "BackwardStrategy":
        return cls("vanilla", PathSpec("fp"), PathSpec("fp"))

    @classmethod
    def naive_quant(cls, bits: int = 4) -> "BackwardStrategy":
        return cls(f"int{bits}", PathSpec("quant", bits), PathSpec("quant", bits))

    @classmethod
    def hq(cls, bits_gx: int = 4, bits_gw: int = 4, block: int = DEFAULT_BLOCK) -> "BackwardStrategy":
        plan = HadamardPlan(block_size=block, basis_indices=tuple(range(block)))
        return cls("hq", PathSpec("ht_quant", bits_gx), PathSpec("ht_quant", bits_gw), plan)

    @classmethod
    def lbp_wht(cls, rank: int = DEFAULT_RANK, block: int = DEFAULT_BLOCK) -> "BackwardStrategy":
        plan = HadamardPlan(block_size=block, basis_indices=lowest_sequency_bases(block, rank))
        return cls("lbp-wht", PathSpec("lowrank"), PathSpec("lowrank"), plan)

    @classmethod
    def hlq(cls, bits_gx: int = 4, bits_gw: int = 8, rank: int = DEFAULT_RANK,
            block: int = DEFAULT_BLOCK) -> "BackwardStrategy":
        plan = HadamardPlan(block_size=block, basis_indices=lowest_sequency_bases(block, rank))
        return cls("hlq", PathSpec("ht_quant", bits_gx), PathSpec("lowrank_quant", bits_gw), plan)

    def float_pipeline(self) -> "BackwardStrategy":
        """Quantizers removed, transforms and rank kept (backprop.py:120-128)."""
        return replace(self, name=f"{self.name}[float]",
                       grad_input_path=replace(self.grad_input_path, bits=None),
                       grad_weight_path=replace(self.grad_weight_path, bits=None))

    def debug_exact(self) -> "BackwardStrategy":
        """No quantization, full rank: reproduces the vanilla backward (backprop.py:130-137)."""
        return replace(self.float_pipeline(), name=f"{self.name}[exact]",
                       plan=self.plan.with_rank(self.plan.block_size))

    @property
    def is_hlq(self) -> bool:
        """The combined scheme the fused training kernels implement."""
        return (self.grad_input_path.mode == "ht_quant" and self.grad_input_path.bits is not None
                and self.grad_weight_path.mode == "lowrank_quant" and self.grad_weight_path.bits is not None)

    def with_warmup_bits(self, bits: int = 8) -> "BackwardStrategy":
        def widen(spec: PathSpec) -> PathSpec:
            return spec if spec.bits is None else replace(spec, bits=bits)
        return replace(self, name=f"{self.name}[warmup-int{bits}]",
                       grad_input_path=widen(self.grad_input_path),
                       grad_weight_path=widen(self.grad_weight_path))

    def with_plan(self, plan: HadamardPlan) -> "BackwardStrategy":
        return replace(self, plan=plan)

    @property
    def uses_compressed_activation(self) -> bool:
        return self.grad_weight_path.mode == "lowrank_quant" and self.store_compressed


@dataclass(frozen=True)
class QuantizedTensor:
    """int8 codes (kernel layout) + bit width + per-tensor fp32 scale on the device."""

    payload: torch.Tensor
    bits: int
    scale: torch.Tensor
    per_axis: int | None = None

    @property
    def qmax(self) -> int:
        return (1 << (self.bits - 1)) - 1


@dataclass(frozen=True)
class ACBPActivation:
    """Forward-time compressed activation (backprop.py:158-176).

    ``quantized.payload`` is (rows, ld) int8, K-major: rows = I (token axis) or
    L*I (batch axis, row l*I + i); the first ``k`` codes of each row are valid.
    """

    quantized: QuantizedTensor
    orig_shape: tuple
    axis: int
    plan: HadamardPlan
    k: int

    @property
    def payload_nbytes(self) -> int:
        n = self.k * self.quantized.payload.shape[0]
        return n if self.quantized.bits == 8 else (n + 1) // 2

    def reference_payload(self) -> torch.Tensor:
        """The payload in the reference's (K_ref, I) layout (backprop.py:383-385)."""
        B, L, I = self.orig_shape
        p = self.quantized.payload[:, : self.k]
        if self.axis == 1:
            return p.t().contiguous()
        return p.reshape(L, I, self.k).permute(2, 0, 1).reshape(self.k * L, I).contiguous()


def ht_axis_for(B: int, L: int, block: int, pad_small_axes: bool = False) -> int:
    """backprop.py:179-190."""
    if L >= block:
        return 1
    if B >= block:
        return 0
    if not pad_small_axes:
        raise DimensionError(
            f"both L={L} and B={B} are below the block size {block}; set pad_small_axes to zero-pad")
    return 1 if L >= B else 0


def _check_rng(rng):
    if rng is not None and not (hasattr(rng, "seed") and hasattr(rng, "counter")):
        raise ParameterError("rng must be an RngState (seed, counter), e.g. paper_2406_15102_b200.RngState")


def _as3(t: torch.Tensor, what: str) -> torch.Tensor:
    if t.dim() != 3:
        raise DimensionError(f"expected {what} (B,L,C), got {tuple(t.shape)}")
    return t


def _proj_view(B: int, L: int, C: int, axis: int):
    """(segs, rows, cols, ld_src, seg_src) of the projection along `axis`."""
    if axis == 1:
        return B, L, C, C, L * C
    return 1, B, L * C, L * C, B * L * C


def acbp_compress(x: torch.Tensor, plan: HadamardPlan, bits: int = 8, rng=None,
                  pad_small_axes: bool = False, check_finite: bool = True) -> ACBPActivation:
    """backprop.py:373-385 on the GPU: project X along ht_axis_for's axis,
    quantize (int8 by default), keep only the payload."""
    _check_rng(rng)
    x = _as3(x, "x")
    B, L, I = x.shape
    axis = ht_axis_for(B, L, plan.block_size, pad_small_axes)
    segs, rows, cols, ld_src, seg_src = _proj_view(B, L, I, axis)
    if rng is not None:
        # reference quantizes proj (K, I) / (Kb, L, I) in C order: index k*cols + c
        seed, ctr = site_key(rng, TAG_GW_RIGHT)
        codes, scale, amax, k = ops.quant_stochastic(x, segs, rows, cols, ld_src, seg_src, False,
                                                     plan.gpu_bitmap(), bits, seed, ctr, index_kind=1)
    else:
        codes, k, scale, amax = ops.quant_proj_rows(x, segs, rows, cols, plan.gpu_bitmap(), bits,
                                                    ld_src, seg_src)
    if check_finite:
        ops.check_finite(amax)
    q = QuantizedTensor(payload=codes, bits=bits, scale=scale)
    return ACBPActivation(quantized=q, orig_shape=(B, L, I), axis=axis, plan=plan, k=k)


def hq_grad_input(gy: torch.Tensor, w: torch.Tensor, bits: int | None, rng=None,
                  block: int = DEFAULT_BLOCK, out_dtype=torch.float32, exact: bool = True,
                  check_finite: bool = True, stages: dict | None = None) -> torch.Tensor:
    """backprop.py:350-370: dX = deq(Q(HT_O(gy)) . Q(HT_O(W))), full rank, no inverse HT."""
    _check_rng(rng)
    if gy.dim() != 3 or w.dim() != 2:
        raise DimensionError(f"expected gy (B,L,O) and w (O,I), got {tuple(gy.shape)}, {tuple(w.shape)}")
    if gy.shape[2] != w.shape[0]:
        raise DimensionError(f"output channels differ: gy {tuple(gy.shape)} vs w {tuple(w.shape)}")
    if block != 16:
        raise ParameterError(f"the B200 kernels implement block 16 only, got {block}")
    B, L, O = gy.shape
    I = w.shape[1]
    if bits is None:
        # transforms only, float GEMM (backprop.py:364-366): ghat @ what == gy @ w up to roundoff
        ghat = _block_f32(gy.reshape(B * L, O), along_cols=True)
        what = _block_f32(w, along_cols=False)
        return (ghat @ what).reshape(B, L, I)
    w32 = w if w.dtype == torch.float32 else w.float()
    if rng is not None:
        seed, ctr = site_key(rng, TAG_GX_LEFT)
        g2 = gy.reshape(B * L, O).contiguous()
        cg, sg, ag = ops.quant_stochastic(g2, 1, B * L, O, O, B * L * O, True, 0xFFFF, bits, seed, ctr)
        seed, ctr = site_key(rng, TAG_GX_RIGHT)
        cw, sw, aw, kw = ops.quant_stochastic(w32.contiguous(), 1, O, I, I, O * I, False, 0xFFFF, bits, seed,
                                              ctr, index_kind=1)
    else:
        cg, sg, ag = ops.quant_ht_cols(gy.reshape(B * L, O), bits)
        cw, kw, sw, aw = ops.quant_proj_rows(w32, 1, O, I, 0xFFFF, bits)
    if check_finite:
        ops.check_finite(ag, aw)
    out, acc = ops.gemm_i8(cg, cw, B * L, I, ops.pad16(O), bits, bits, sg, sw, 1.0, exact=exact,
                           out_dtype=out_dtype, want_acc=stages is not None)
    if stages is not None:
        stages.update(gx_codes_g=cg[:, :ops.pad16(O)], gx_scale_g=sg, gx_codes_w=cw[:, :kw].t(),
                      gx_scale_w=sw, gx_acc=acc)
    return out.reshape(B, L, I)


def _gy_projection(gy: torch.Tensor, axis: int, plan: HadamardPlan, bits: int):
    B, L, O = gy.shape
    segs, rows, cols, ld_src, seg_src = _proj_view(B, L, O, axis)
    return ops.quant_proj_rows(gy, segs, rows, cols, plan.gpu_bitmap(), bits, ld_src, seg_src)


def hlq_grad_weight(acbp: ACBPActivation, gy: torch.Tensor, bits: int = 8, rng=None,
                    extra_scale: float | None = None, out_dtype=torch.float32, exact: bool = True,
                    check_finite: bool = True, stages: dict | None = None) -> torch.Tensor:
    """backprop.py:388-410: project gy onto the ACBP bases, quantize, int8 GEMM
    against the stored payload, dequantize with s_g * s_x * extra (1/B by default)."""
    _check_rng(rng)
    B, L, I = acbp.orig_shape
    if gy.dim() != 3 or gy.shape[0] != B or gy.shape[1] != L:
        raise StateError(f"gy shape {tuple(gy.shape)} does not match the compressed activation ({B}, {L}, ...)")
    if acbp.quantized.bits != bits:
        raise StateError(f"compressed activation is {acbp.quantized.bits}-bit but backward wants {bits}-bit")
    O = gy.shape[2]
    if rng is not None:
        # the reference quantizes gy2.T: (O, K) for tokens / L == 1, (O, Kb*L) for the batch axis
        seed, ctr = site_key(rng, TAG_GW_LEFT)
        segs, rows, cols, ld_src, seg_src = _proj_view(B, L, O, acbp.axis)
        kind = 2 if (acbp.axis == 0 and L > 1) else 0
        cg, sg, ag, k = ops.quant_stochastic(gy.contiguous(), segs, rows, cols, ld_src, seg_src, False,
                                             acbp.plan.gpu_bitmap(), bits, seed, ctr, index_kind=kind,
                                             l2=L, o2=O)
    else:
        cg, k, sg, ag = _gy_projection(gy, acbp.axis, acbp.plan, bits)
    if k != acbp.k:
        raise StateError("projected extents differ between forward and backward; the plans do not match")
    if check_finite:
        ops.check_finite(ag)
    extra = 1.0 / B if extra_scale is None else extra_scale
    groups = L if acbp.axis == 0 else 1
    xp = acbp.quantized.payload
    out, acc = ops.gemm_i8(cg, xp, O, I, k, bits, bits, sg, acbp.quantized.scale, extra,
                           exact=exact, out_dtype=out_dtype, want_acc=stages is not None,
                           groups=groups, a_gstride=cg.stride(0) * O, b_gstride=xp.stride(0) * I)
    if stages is not None:
        stages.update(gw_codes_g=cg[:, :k], gw_scale_g=sg, gw_acc=acc)
    return out


def dual_ok(B: int, L: int, axis: int) -> bool:
    """The fused gy transform needs the projection view's rows to be the HT
    view's rows: projection along tokens, or along the batch with L == 1."""
    return axis == 1 or L == 1


def hlq_pair(acbp: ACBPActivation, w: torch.Tensor, gy: torch.Tensor, bits_gx: int, bits_gw: int,
             extra_scale: float, exact: bool = True, gx_dtype=torch.float32,
             check_finite: bool = True, stages: dict | None = None):
    """Both HLQ products with ONE fused transform of gy (two passes instead of
    four): returns (gx (B, L, I), gw (O, I)).  Same numerics as calling
    hlq_grad_weight and hq_grad_input separately."""
    B, L, I = acbp.orig_shape
    O = gy.shape[2]
    if acbp.quantized.bits != bits_gw:
        raise StateError(f"compressed activation is {acbp.quantized.bits}-bit but backward wants {bits_gw}-bit")
    segs, rows, cols, ld_src, seg_src = _proj_view(B, L, O, acbp.axis)
    cgx, sgx, cgw, k, sgw, st = ops.quant_dual(gy, segs, rows, cols, acbp.plan.gpu_bitmap(),
                                               bits_gx, bits_gw, ld_src, seg_src)
    if k != acbp.k:
        raise StateError("projected extents differ between forward and backward; the plans do not match")
    w32 = w if w.dtype == torch.float32 else w.float()
    cw, kw, sw, aw = ops.quant_proj_rows(w32, 1, O, I, 0xFFFF, bits_gx)
    if check_finite:
        ops.check_finite(st[0:1], st[2:3], aw)
    xp = acbp.quantized.payload
    want = stages is not None
    gw, accw = ops.gemm_i8(cgw, xp, O, I, k, bits_gw, bits_gw, sgw, acbp.quantized.scale, extra_scale,
                           exact=exact, want_acc=want)
    gx, accx = ops.gemm_i8(cgx, cw, B * L, I, ops.pad16(O), bits_gx, bits_gx, sgx, sw, 1.0,
                           exact=exact, out_dtype=gx_dtype, want_acc=want)
    if want:
        stages.update(gx_codes_g=cgx, gx_scale_g=sgx, gx_codes_w=cw[:, :kw].t(), gx_scale_w=sw,
                      gx_acc=accx, gw_codes_g=cgw[:, :k], gw_scale_g=sgw, gw_acc=accw)
    return gx.reshape(B, L, I), gw


def _vanilla_gx(gy, w):
    B, L, O = gy.shape
    return (gy.reshape(-1, O).float() @ w.float()).reshape(B, L, -1)


def _vanilla_gw(x, gy, extra):
    B, L, I = x.shape
    return (gy.reshape(-1, gy.shape[2]).float().t() @ x.reshape(-1, I).float()) * extra


# ---------------------------------------------------------------------------
# baseline strategies: naive quant, HQ on dW, LBP-WHT and
# the bits=None float pipelines, on the hlq_xform_* kernels; float GEMMs are
# cuBLAS fp32 (torch matmul; TF32 stays off unless the caller enables it)
# ---------------------------------------------------------------------------

def _block_f32(m: torch.Tensor, along_cols: bool) -> torch.Tensor:
    """_block_axis of a 2-D (R, C) matrix in float32: along its columns axis
    (-> (R, pad16(C))) or its rows axis (-> (pad16(R), C))."""
    R, C = m.shape
    m = m.contiguous()
    if along_cols:
        out = torch.empty((R, ops.pad16(C)), dtype=torch.float32, device=m.device)
        return ops.xform_project(m, 1, C, R, (0, 1, C), 0xFFFF, out, (0, 1, out.stride(0)))
    out = torch.empty((ops.pad16(R), C), dtype=torch.float32, device=m.device)
    return ops.xform_project(m, 1, R, C, (0, C, 1), 0xFFFF, out, (0, C, 1))


def _project_f32(t: torch.Tensor, axis: int, bitmap: int) -> torch.Tensor:
    """_project_axis (backprop.py:223-234) of (B, L, C) along `axis` in float32,
    in the reference's shape: (B, K, C) for axis 1, (Kb, L, C) for axis 0."""
    B, L, C = t.shape
    segs, rows, cols, ld_src, seg_src = _proj_view(B, L, C, axis)
    kps = ((rows + 15) // 16) * bin(bitmap).count("1")
    out = torch.empty((segs, kps, cols), dtype=torch.float32, device=t.device)
    ops.xform_project(t.contiguous(), segs, rows, cols, (seg_src, ld_src, 1), bitmap, out, (kps * cols, cols, 1))
    return out if axis == 1 else out.reshape(kps, L, C)


def _unproject_f32(coeff: torch.Tensor, axis: int, bitmap: int, B: int, L: int, C: int) -> torch.Tensor:
    """_unproject_axis (backprop.py:237-249) back to (B, L, C)."""
    segs, rows, cols, ld_src, seg_src = _proj_view(B, L, C, axis)
    kps = ((rows + 15) // 16) * bin(bitmap).count("1")
    out = torch.empty((B, L, C), dtype=torch.float32, device=coeff.device)
    return ops.xform_unproject(coeff.contiguous(), segs, rows, cols, (kps * cols, cols, 1), bitmap, out,
                               (seg_src, ld_src, 1))


def _plain_codes(m: torch.Tensor, bits: int, rng, tag: int, contract_rows: bool, ref_transposed: bool = False):
    """_quant of a 2-D (R, C) matrix with no transform (the "quant" mode) as a
    K-major GEMM operand: contracted over C -> codes (R, pad16(C)); over R ->
    codes (C, pad16(R)).  ref_transposed: the reference quantizes m.T (its
    draw index is c*R + r).  Returns (codes, scale, amax_bits)."""
    R, C = m.shape
    m = m.contiguous()
    if contract_rows:
        codes = torch.zeros((C, max(ops.pad16(R), 16)), dtype=torch.int8, device=m.device)
        dst = (0, 1, codes.stride(0))
    else:
        codes = torch.zeros((R, max(ops.pad16(C), 16)), dtype=torch.int8, device=m.device)
        dst = (0, codes.stride(0), 1)
    seed, ctr = site_key(rng, tag) if rng is not None else (None, 0)
    idx = (0, 1, R) if ref_transposed else (0, C, 1)
    scale, amax = ops.xform_quantize(m, 1, R, C, (0, C, 1), 0, codes, dst, bits, seed, ctr, idx)
    return codes, scale, amax


def _naive_gx(gy, w, bits, rng, check_finite=True):
    """backprop.py:301-307: Q(gy (M, O)) . Q(W (O, I)), both quantized directly."""
    B, L, O = gy.shape
    I = w.shape[1]
    cg, sg, ag = _plain_codes(gy.reshape(B * L, O), bits, rng, TAG_GX_LEFT, contract_rows=False)
    cw, sw, aw = _plain_codes(w if w.dtype == torch.float32 else w.float(), bits, rng, TAG_GX_RIGHT,
                              contract_rows=True)
    if check_finite:
        ops.check_finite(ag, aw)
    out, _ = ops.gemm_i8(cg, cw, B * L, I, cg.shape[1], bits, bits, sg, sw, 1.0, exact=True)
    return out.reshape(B, L, I)


def _naive_gw(x, gy, bits, rng, extra, check_finite=True):
    """backprop.py:256-291 with mode "quant": Q(gy2^T (O, K)) . Q(x2 (K, I)), K = B*L."""
    B, L, I = x.shape
    O = gy.shape[2]
    K = B * L
    cg, sg, ag = _plain_codes(gy.reshape(K, O), bits, rng, TAG_GW_LEFT, contract_rows=True, ref_transposed=True)
    cx, sx, ax = _plain_codes(x.reshape(K, I), bits, rng, TAG_GW_RIGHT, contract_rows=True)
    if check_finite:
        ops.check_finite(ag, ax)
    out, _ = ops.gemm_i8(cg, cx, O, I, cg.shape[1], bits, bits, sg, sx, extra, exact=True)
    return out


def _lowrank_gx(gy, w, strategy: BackwardStrategy):
    """backprop.py:310-316: project gy, float GEMM, inverse projection."""
    B, L, O = gy.shape
    I = w.shape[1]
    axis = ht_axis_for(B, L, strategy.plan.block_size, strategy.pad_small_axes)
    bm = strategy.plan.gpu_bitmap()
    ghat = _project_f32(gy, axis, bm)
    gx_hat = (ghat.reshape(-1, O) @ w.float()).reshape(*ghat.shape[:-1], I)
    return _unproject_f32(gx_hat, axis, bm, B, L, I)


def _float_gw(x, gy, plan: HadamardPlan | None, strategy: BackwardStrategy, extra):
    """_gw_operands + the bits=None branch of _gw_from_operands (backprop.py:256-276):
    project x and gy along the token (or batch) axis, float GEMM."""
    B, L, I = x.shape
    O = gy.shape[2]
    if plan is None:
        return _vanilla_gw(x, gy, extra)
    axis = ht_axis_for(B, L, plan.block_size, strategy.pad_small_axes)
    bm = plan.gpu_bitmap()
    x2 = _project_f32(x, axis, bm).reshape(-1, I)
    gy2 = _project_f32(gy, axis, bm).reshape(-1, O)
    return (gy2.t() @ x2) * extra


def _full(plan: HadamardPlan) -> HadamardPlan:
    return plan.with_rank(plan.block_size)


def _grad_input(gy, w, strategy: BackwardStrategy, rng, stages=None):
    """backprop.py:294-316."""
    spec = strategy.grad_input_path
    if spec.mode == "fp" or (spec.mode == "quant" and spec.bits is None):
        return _vanilla_gx(gy, w)
    if spec.mode == "quant":
        return _naive_gx(gy, w, spec.bits, rng)
    if spec.mode == "ht_quant":
        return hq_grad_input(gy, w, spec.bits, rng=rng, block=strategy.plan.block_size, stages=stages)
    return _lowrank_gx(gy, w, strategy)


def _grad_weight(x, gy, strategy: BackwardStrategy, rng, extra):
    """backprop.py:256-291 for the raw-activation modes."""
    spec = strategy.grad_weight_path
    if spec.mode == "fp" or (spec.mode == "quant" and spec.bits is None):
        return _vanilla_gw(x, gy, extra)
    if spec.mode == "quant":
        return _naive_gw(x, gy, spec.bits, rng, extra)
    if spec.bits is None:  # ht_quant / lowrank_quant float pipelines, lowrank
        plan = _full(strategy.plan) if spec.mode == "ht_quant" else strategy.plan
        return _float_gw(x, gy, plan, strategy, extra)
    if spec.mode == "ht_quant":
        # full-rank block transform along the token axis, quantized: the HLQ dW
        # kernels with every basis kept (same tags, same C-order draw indices)
        acbp = acbp_compress(x, _full(strategy.plan), bits=spec.bits, rng=rng,
                             pad_small_axes=strategy.pad_small_axes)
        return hlq_grad_weight(acbp, gy, bits=spec.bits, rng=rng, extra_scale=extra)
    raise ParameterError(f"grad_weight mode {spec.mode!r} needs the compressed activation path")


def strategy_backward(x_or_acbp, w: torch.Tensor, gy: torch.Tensor, strategy: BackwardStrategy,
                      rng=None, stages: dict | None = None, gw_scale: float | None = None) -> GradPair:
    """backprop.py:413-435.  gw_scale replaces the 1/B mean factor of the
    weight gradient (the torch modules pass 1: autograd's gy already has it)."""
    _check_rng(rng)
    if isinstance(x_or_acbp, ACBPActivation):
        acbp = x_or_acbp
        if strategy.grad_weight_path.mode != "lowrank_quant":
            raise StateError(f"strategy {strategy.name!r} expects the raw activation, not a compressed one")
        if (acbp.plan.block_size != strategy.plan.block_size
                or acbp.plan.basis_indices != strategy.plan.basis_indices):
            raise StateError("compressed activation was built with a different plan")
        B, L, I = acbp.orig_shape
        if gy.dim() != 3 or tuple(gy.shape[:2]) != (B, L) or w.shape[1] != I:
            raise DimensionError(f"gy {tuple(gy.shape)} / w {tuple(w.shape)} do not match activation {acbp.orig_shape}")
        bits_gw = strategy.grad_weight_path.bits or 8
        extra = 1.0 / B if gw_scale is None else gw_scale
        if (strategy.grad_input_path.mode == "ht_quant" and strategy.grad_input_path.bits
                and rng is None and dual_ok(B, L, acbp.axis)):
            gx, gw = hlq_pair(acbp, w, gy, strategy.grad_input_path.bits, bits_gw, extra,
                              stages=stages)
            return GradPair(gx, gw)
        gw = hlq_grad_weight(acbp, gy, bits=bits_gw, rng=rng, extra_scale=extra, stages=stages)
        gx = _grad_input(gy, w, strategy, rng, stages)
        return GradPair(gx, gw)
    x = x_or_acbp
    if x.dim() != 3 or gy.dim() != 3 or w.dim() != 2:
        raise DimensionError(
            f"expected x (B,L,I), w (O,I), gy (B,L,O); got {tuple(x.shape)}, {tuple(w.shape)}, {tuple(gy.shape)}")
    B, L, I = x.shape
    O = w.shape[0]
    if w.shape[1] != I:
        raise DimensionError(f"weight {tuple(w.shape)} does not match input channels {I}")
    if tuple(gy.shape) != (B, L, O):
        raise DimensionError(f"gy shape {tuple(gy.shape)} does not match ({B}, {L}, {O})")
    spec = strategy.grad_weight_path
    if spec.mode == "lowrank_quant" and spec.bits is not None:
        # raw branch == ACBP branch bit for bit in pseudo mode (test_backprop.py:338-345)
        acbp = acbp_compress(x, strategy.plan, bits=spec.bits or 8, rng=rng,
                             pad_small_axes=strategy.pad_small_axes)
        if stages is not None:
            stages.update(x_codes=acbp.reference_payload(), x_scale=acbp.quantized.scale, axis=acbp.axis)
        return strategy_backward(acbp, w, gy, strategy, rng=rng, stages=stages, gw_scale=gw_scale)
    gx = _grad_input(gy, w, strategy, rng, stages)
    gw = _grad_weight(x, gy, strategy, rng, 1.0 / B if gw_scale is None else gw_scale)
    return GradPair(gx, gw)


def vanilla_backward(x: torch.Tensor, w: torch.Tensor, gy: torch.Tensor) -> GradPair:
    """backprop.py:326-331: the exact chain rule (float32 GEMMs)."""
    return strategy_backward(x, w, gy, BackwardStrategy.vanilla())


def naive_quant_backward(x: torch.Tensor, w: torch.Tensor, gy: torch.Tensor, bits: int, rng=None) -> GradPair:
    """backprop.py:334-337: both products on directly quantized operands."""
    return strategy_backward(x, w, gy, BackwardStrategy.naive_quant(bits), rng=rng)


def lbp_wht_backward(x: torch.Tensor, w: torch.Tensor, gy: torch.Tensor, plan: HadamardPlan,
                     pad_small_axes: bool = False) -> GradPair:
    """backprop.py:340-347: low-rank basis truncation on both paths (float GEMMs)."""
    if plan.full_rank:
        raise ParameterError("plan is full-rank; low-rank backward needs rank < block size")
    strategy = BackwardStrategy("lbp-wht", PathSpec("lowrank"), PathSpec("lowrank"), plan=plan,
                                pad_small_axes=pad_small_axes)
    return strategy_backward(x, w, gy, strategy)


def hlq_backward(x_or_acbp, w: torch.Tensor, gy: torch.Tensor,
                 strategy: BackwardStrategy | None = None, rng=None,
                 stages: dict | None = None) -> GradPair:
    """backprop.py:438-447: int4 HQ input gradient + int8 low-rank weight gradient."""
    strategy = strategy or BackwardStrategy.hlq()
    if strategy.grad_weight_path.mode != "lowrank_quant" or strategy.grad_input_path.mode != "ht_quant":
        raise ParameterError(f"hlq_backward requires the combined strategy, got {strategy.name!r}")
    return strategy_backward(x_or_acbp, w, gy, strategy, rng=rng, stages=stages)
