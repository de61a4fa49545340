"""CPU oracle for the HLQ backward path -- TEST INFRASTRUCTURE, NOT PRODUCT CODE.

This module is a numpy restatement of the reference's algorithm for the one hot
path this repository accelerates (HLQ backward for Linear / Conv2d plus the
forward-time ACBP compression).  It exists only to *check* the CUDA path:

* only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
  ``cpu_baseline`` / ``--impl reference`` leg may import it;
* nothing under ``paper_2406_15102_b200/`` imports it -- the product path has
  no CPU fallback and fails loudly when its CUDA library is missing.

Parity pinning: every function below is validated bit-for-bit against golden
vectors produced by the reference itself (``tests/golden/make_golden.py``
imports ``/root/reference/pkg/src/hlq`` in the build container and stores the
outputs under ``tests/golden/*.npz``; ``tests/test_oracle_golden.py`` checks
this module against them).

Reference anchors (paths relative to ``/root/reference/pkg/src/hlq``):
  hadamard.py:24-49    sequency ordering / default basis sets
  hadamard.py:121-134  orthonormal radix-2 FWHT, stage order h = 1, 2, 4, ...
  tensor.py:91-95,125-135  zero padding to a block multiple
  backprop.py:179-190  projection-axis rule
  backprop.py:212-234  block transform / low-rank projection along one axis
  quantize.py:94-100   per-tensor symmetric scale
  quantize.py:128-145  pseudo-stochastic rounding (low 11 bits as the draw)
  quantize.py:26-59,114-125  RngState (splitmix64 splits, Philox4x64 draws) and
                       true stochastic rounding; backprop.py:42-43,206-209 tags
  quantize.py:152-187  exact integer GEMM + fp64 dequant epilogue
  backprop.py:350-447  hq_grad_input / acbp_compress / hlq_grad_weight / hlq_backward
  backprop.py:237-347  baseline strategies (naive quant, HQ, LBP-WHT, float pipelines)
  harness/layers.py:96-158  conv lowering (im2col / col2im)
"""
from __future__ import annotations

import numpy as np

F32 = np.float32
QMAX = {4: 7, 8: 127}


class OracleError(ValueError):
    pass


# ---------------------------------------------------------------------------
# basis sets (hadamard.py:24-49)
# ---------------------------------------------------------------------------

def sequency_of_row(i: int, n: int) -> int:
    """Sign changes of natural-order Walsh row ``i``: Gray-decode of the
    bit-reversed index (hadamard.py:34-43)."""
    k = n.bit_length() - 1
    rev = 0
    for b in range(k):
        if i >> b & 1:
            rev |= 1 << (k - 1 - b)
    g, shift = rev, 1
    while shift < 32:
        g ^= g >> shift
        shift <<= 1
    return g


def lowest_sequency_bases(n: int, r: int) -> tuple:
    order = sorted(range(n), key=lambda i: (sequency_of_row(i, n), i))
    return tuple(sorted(order[:r]))


# ---------------------------------------------------------------------------
# transforms (hadamard.py:121-134, backprop.py:212-234)
# ---------------------------------------------------------------------------

def fwht_blocks(a: np.ndarray) -> np.ndarray:
    """Orthonormal FWHT over the last axis (length n, power of two), fp32.

    Stage order h = 1, 2, 4, ... with (lower, upper) = (a + b, a - b) for
    every pair (i, i + h), i & h == 0, then one multiply by fp32(1/sqrt(n)).
    The stage order is part of the bit-exact contract (hadamard.py:125-133).
    """
    x = np.array(a, dtype=F32, copy=True)
    n = x.shape[-1]
    h = 1
    while h < n:
        lo = np.array([i for i in range(n) if not i & h])
        hi = lo + h
        a_, b_ = x[..., lo], x[..., hi]
        x[..., lo] = a_ + b_
        x[..., hi] = a_ - b_
        h <<= 1
    return x * F32(1.0 / np.sqrt(n))


def pad_to(a: np.ndarray, axis: int, n: int) -> np.ndarray:
    ext = a.shape[axis]
    tgt = -(-ext // n) * n
    if tgt == ext:
        return a
    widths = [(0, 0)] * a.ndim
    widths[axis] = (0, tgt - ext)
    return np.pad(a, widths)


def transform_axis(a: np.ndarray, axis: int, n: int, bases=None) -> np.ndarray:
    """Pad ``axis`` to a multiple of n, block-FWHT it, and (when ``bases`` is
    given) keep only those coefficient rows of every block."""
    p = pad_to(np.asarray(a, dtype=F32), axis, n)
    m = np.moveaxis(p, axis, -1)
    lead = m.shape[:-1]
    nb = m.shape[-1] // n
    c = fwht_blocks(m.reshape(*lead, nb, n))
    if bases is not None and len(bases) != n:
        c = c[..., list(bases)]
    out = c.reshape(*lead, nb * c.shape[-1])
    return np.ascontiguousarray(np.moveaxis(out, -1, axis))


def proj_axis_rule(B: int, L: int, n: int, pad_small_axes: bool = False) -> int:
    """backprop.py:179-190: L when L >= n, else B when B >= n."""
    if L >= n:
        return 1
    if B >= n:
        return 0
    if not pad_small_axes:
        raise OracleError(f"L={L} and B={B} both below block {n}")
    return 1 if L >= B else 0


# ---------------------------------------------------------------------------
# quantizer + integer GEMM (quantize.py:94-187)
# ---------------------------------------------------------------------------

def quantize(v: np.ndarray, bits: int):
    """Per-tensor symmetric pseudo-stochastic quantizer -> (int8 codes, f32 scale)."""
    qmax = QMAX[bits]
    v = np.ascontiguousarray(v, dtype=F32)
    if not np.isfinite(v).all():
        raise OracleError("non-finite input")
    amax = F32(np.abs(v).max()) if v.size else F32(0)
    scale = F32(amax / F32(qmax))
    if scale == 0:
        scale = F32(1.0)
    q = v / scale
    lo = np.floor(q)
    draw = (v.view(np.uint32) & np.uint32(0x7FF)).astype(F32)
    bump = ((q - lo) * F32(2048.0)) > draw
    codes = np.clip(lo + bump.astype(F32), -qmax, qmax).astype(np.int8)
    return codes, scale


def quantize_with_amax(v: np.ndarray, bits: int, amax) -> tuple:
    """quantize() with the per-tensor amax supplied (e.g. reduced over data-
    parallel shards): the codes the single-process quantizer produces for this
    slice of a larger tensor."""
    qmax = QMAX[bits]
    v = np.ascontiguousarray(v, dtype=F32)
    scale = F32(F32(amax) / F32(qmax))
    if scale == 0:
        scale = F32(1.0)
    q = v / scale
    lo = np.floor(q)
    draw = (v.view(np.uint32) & np.uint32(0x7FF)).astype(F32)
    bump = ((q - lo) * F32(2048.0)) > draw
    return np.clip(lo + bump.astype(F32), -qmax, qmax).astype(np.int8), scale


# ---------------------------------------------------------------------------
# true stochastic rounding (quantize.py:26-59,114-125; backprop.py:42-43,206-209)
# ---------------------------------------------------------------------------

TAG_GX_LEFT, TAG_GX_RIGHT, TAG_GW_LEFT, TAG_GW_RIGHT = 11, 12, 21, 22
_M64 = (1 << 64) - 1


def splitmix64(x: int) -> int:
    x = (x + 0x9E3779B97F4A7C15) & _M64
    x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & _M64
    x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & _M64
    return (x ^ (x >> 31)) & _M64


def split_seed(seed: int, *path: int) -> int:
    """RngState(seed).split(*path).seed (quantize.py:48-52)."""
    key = int(seed) & _M64
    for p in path:
        key = splitmix64(key ^ splitmix64(int(p) & _M64))
    return key


def uniform(seed: int, counter: int, shape) -> np.ndarray:
    """RngState(seed, counter).uniform(shape): numpy's Philox4x64-10 keyed
    [seed, counter], float64 draws in C order (quantize.py:54-59)."""
    key = np.array([int(seed) & _M64, int(counter) & _M64], dtype=np.uint64)
    return np.random.Generator(np.random.Philox(key=key)).random(size=shape)


def quantize_stochastic(v: np.ndarray, bits: int, seed: int):
    """quant_stochastic(v, bits, RngState(seed)) (quantize.py:114-125):
    up = f64(q - floor(q)) > U.  -> (int8 codes, f32 scale)."""
    qmax = QMAX[bits]
    v = np.ascontiguousarray(v, dtype=F32)
    if not np.isfinite(v).all():
        raise OracleError("non-finite input")
    amax = F32(np.abs(v).max()) if v.size else F32(0)
    scale = F32(amax / F32(qmax))
    if scale == 0:
        scale = F32(1.0)
    q = v / scale
    lo = np.floor(q)
    up = (q - lo) > uniform(seed, 0, v.shape)
    codes = np.clip(lo + up.astype(F32), -qmax, qmax).astype(np.int8)
    return codes, scale


def _q(v: np.ndarray, bits: int, rng_seed, tag: int):
    """_quant (backprop.py:206-209): pseudo when rng is None, else stochastic
    on the tag's split stream."""
    if rng_seed is None:
        return quantize(v, bits)
    return quantize_stochastic(v, bits, split_seed(rng_seed, tag))


def int_gemm(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    """Exact sum of int8 products; fp64 BLAS is exact below 2**53."""
    return (a.astype(np.float64) @ b.astype(np.float64)).astype(np.int64)


def dequant(acc: np.ndarray, sa, sb, extra: float = 1.0) -> np.ndarray:
    comb = F32(F32(sa) * F32(sb))
    return (acc.astype(np.float64) * (np.float64(comb) * float(extra))).astype(F32)


# ---------------------------------------------------------------------------
# the HLQ path (backprop.py:350-447)
# ---------------------------------------------------------------------------

def hq_grad_input(gy3: np.ndarray, w: np.ndarray, bits: int = 4, n: int = 16,
                  stages: dict | None = None, rng: int | None = None) -> np.ndarray:
    """rng: the RngState seed (counter 0) for true stochastic rounding, or None."""
    B, L, O = gy3.shape
    I = w.shape[1]
    ghat = transform_axis(gy3, 2, n).reshape(B * L, -1)
    what = transform_axis(w, 0, n)
    cg, sg = _q(ghat, bits, rng, TAG_GX_LEFT)
    cw, sw = _q(what, bits, rng, TAG_GX_RIGHT)
    acc = int_gemm(cg, cw)
    out = dequant(acc, sg, sw).reshape(B, L, I)
    if stages is not None:
        stages.update(gx_codes_g=cg, gx_scale_g=sg, gx_codes_w=cw, gx_scale_w=sw, gx_acc=acc)
    return out


def acbp_compress(x3: np.ndarray, bases, bits: int = 8, n: int = 16,
                  pad_small_axes: bool = False, rng: int | None = None):
    """Forward-time projection + quantization of X -> (payload (K, I), scale, axis)."""
    B, L, I = x3.shape
    axis = proj_axis_rule(B, L, n, pad_small_axes)
    proj = transform_axis(x3, axis, n, bases)
    codes, scale = _q(proj, bits, rng, TAG_GW_RIGHT)
    return codes.reshape(-1, I), scale, axis


def hlq_grad_weight(payload: np.ndarray, x_scale, axis: int, gy3: np.ndarray,
                    bases, bits: int = 8, n: int = 16, extra: float | None = None,
                    stages: dict | None = None, rng: int | None = None) -> np.ndarray:
    B, L, O = gy3.shape
    gproj = transform_axis(gy3, axis, n, bases).reshape(-1, O)
    if gproj.shape[0] != payload.shape[0]:
        raise OracleError("projected extents differ")
    cg, sg = _q(np.ascontiguousarray(gproj.T), bits, rng, TAG_GW_LEFT)
    acc = int_gemm(cg, payload)
    out = dequant(acc, sg, x_scale, 1.0 / B if extra is None else extra)
    if stages is not None:
        stages.update(gw_codes_g=cg, gw_scale_g=sg, gw_acc=acc)
    return out


def hlq_backward(x3: np.ndarray, w: np.ndarray, gy3: np.ndarray, rank: int = 8,
                 bits_gx: int = 4, bits_gw: int = 8, n: int = 16, bases=None,
                 pad_small_axes: bool = False, extra: float | None = None,
                 stages: dict | None = None, rng: int | None = None):
    """ACBP branch of strategy_backward (backprop.py:416-430): gw then gx.
    rng: RngState seed for true stochastic rounding (every site splits it by
    its tag, so forward ACBP and backward draw independent streams)."""
    bases = lowest_sequency_bases(n, rank) if bases is None else tuple(bases)
    payload, sx, axis = acbp_compress(x3, bases, bits_gw, n, pad_small_axes, rng)
    if stages is not None:
        stages.update(x_codes=payload, x_scale=sx, axis=axis)
    gw = hlq_grad_weight(payload, sx, axis, gy3, bases, bits_gw, n, extra, stages, rng)
    gx = hq_grad_input(gy3, w, bits_gx, n, stages, rng)
    return gx, gw


# ---------------------------------------------------------------------------
# baseline strategies (backprop.py:91-155, 237-347)
# ---------------------------------------------------------------------------

def untransform_axis(c: np.ndarray, axis: int, n: int, bases, extent: int) -> np.ndarray:
    """_unproject_axis (backprop.py:237-249): scatter the kept coefficients of
    every block into n slots (zeros elsewhere), FWHT (orthonormal, its own
    inverse), crop ``axis`` back to ``extent``."""
    m = np.moveaxis(np.asarray(c, dtype=F32), axis, -1)
    r = len(bases)
    nb = m.shape[-1] // r
    full = np.zeros((*m.shape[:-1], nb, n), dtype=F32)
    full[..., list(bases)] = m.reshape(*m.shape[:-1], nb, r)
    out = fwht_blocks(full).reshape(*m.shape[:-1], nb * n)[..., :extent]
    return np.ascontiguousarray(np.moveaxis(out, -1, axis))


def _float_gemm(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    return (a.astype(F32) @ b.astype(F32)).astype(F32)


def strategy_backward(x3: np.ndarray, w: np.ndarray, gy3: np.ndarray, gx_mode: str, gx_bits,
                      gw_mode: str, gw_bits, bases, n: int = 16, pad_small_axes: bool = False,
                      rng: int | None = None):
    """Raw-activation branch of strategy_backward (backprop.py:431-435) for every
    gradient mode: fp, quant (direct), ht_quant (full-rank block transform),
    lowrank (projection, float GEMM, dX unprojected), lowrank_quant (HLQ);
    bits None = the float pipeline of a quantizing mode.  Returns (gx, gw)."""
    B, L, I = x3.shape
    O = w.shape[0]
    bases = tuple(bases)
    full = tuple(range(n))
    # grad_input (backprop.py:294-316)
    if gx_mode == "fp" or (gx_mode == "quant" and gx_bits is None):
        gx = _float_gemm(gy3.reshape(-1, O), w).reshape(B, L, I)
    elif gx_mode == "quant":
        cg, sg = _q(gy3.reshape(-1, O), gx_bits, rng, TAG_GX_LEFT)
        cw, sw = _q(w, gx_bits, rng, TAG_GX_RIGHT)
        gx = dequant(int_gemm(cg, cw), sg, sw).reshape(B, L, I)
    elif gx_mode == "ht_quant":
        if gx_bits is None:
            ghat = transform_axis(gy3, 2, n).reshape(B * L, -1)
            gx = _float_gemm(ghat, transform_axis(w, 0, n)).reshape(B, L, I)
        else:
            gx = hq_grad_input(gy3, w, gx_bits, n, rng=rng)
    elif gx_mode == "lowrank":
        axis = proj_axis_rule(B, L, n, pad_small_axes)
        ghat = transform_axis(gy3, axis, n, bases)
        gxh = _float_gemm(ghat.reshape(-1, O), w).reshape(*ghat.shape[:-1], I)
        gx = untransform_axis(gxh, axis, n, bases, gy3.shape[axis])
    else:
        raise OracleError(f"unknown grad_input mode {gx_mode!r}")
    # grad_weight (backprop.py:256-291)
    inv_b = F32(1.0 / B)
    if gw_mode == "lowrank_quant" and gw_bits is not None:
        payload, sx, axis = acbp_compress(x3, bases, gw_bits, n, pad_small_axes, rng)
        return gx, hlq_grad_weight(payload, sx, axis, gy3, bases, gw_bits, n, rng=rng)
    if gw_mode in ("ht_quant", "lowrank", "lowrank_quant"):
        axis = proj_axis_rule(B, L, n, pad_small_axes)
        keep = full if gw_mode == "ht_quant" else bases
        x2 = transform_axis(x3, axis, n, keep).reshape(-1, I)
        g2 = transform_axis(gy3, axis, n, keep).reshape(-1, O)
    elif gw_mode in ("fp", "quant"):
        x2, g2 = x3.reshape(-1, I), gy3.reshape(-1, O)
    else:
        raise OracleError(f"unknown grad_weight mode {gw_mode!r}")
    if gw_mode in ("fp", "lowrank") or gw_bits is None:
        return gx, (_float_gemm(np.ascontiguousarray(g2.T), x2) * inv_b).astype(F32)
    cg, sg = _q(np.ascontiguousarray(g2.T), gw_bits, rng, TAG_GW_LEFT)
    cx, sx = _q(np.ascontiguousarray(x2), gw_bits, rng, TAG_GW_RIGHT)
    return gx, dequant(int_gemm(cg, cx), sg, sx, 1.0 / B)


# ---------------------------------------------------------------------------
# calibrated basis selection (harness/train.py:128-134, hadamard.py:174-188)
# ---------------------------------------------------------------------------

def basis_energy(gy3: np.ndarray, axis: int, n: int = 16) -> np.ndarray:
    """_basis_energy: per-block |coefficient| matrix (num_blocks_total, n)."""
    moved = np.moveaxis(pad_to(gy3, axis, n), axis, -1)
    blocks = moved.shape[-1] // n
    coeffs = fwht_blocks(np.ascontiguousarray(moved).reshape(*moved.shape[:-1], blocks, n))
    return np.abs(coeffs).reshape(-1, n)


def select_bases(energy: np.ndarray, rank: int) -> tuple:
    means = np.abs(energy).mean(axis=0)
    order = np.argsort(-means, kind="stable")
    return tuple(sorted(int(i) for i in order[:rank]))


# ---------------------------------------------------------------------------
# ACBP container (acbp.py:3-96); CRC32 = zlib's (stdlib), the same function
# the reference calls
# ---------------------------------------------------------------------------

def acbp_container(payload_ref: np.ndarray, bits: int, block: int, bases, B: int, L: int, I: int,
                   scale) -> bytes:
    """acbp_pack: header, scale, payload (C order; int4 two per byte, low
    nibble first, zero high nibble when odd), CRC32 of every prior byte."""
    import struct
    import zlib
    bitmap = 0
    for b in bases:
        bitmap |= 1 << int(b)
    out = bytearray(struct.pack("<4sHBBHHB", b"ACBP", 1, bits, block, len(bases), bitmap, 3))
    out += struct.pack("<3I", B, L, I) + struct.pack("<I", 1) + struct.pack("<f", float(np.float32(scale)))
    flat = np.ascontiguousarray(payload_ref).reshape(-1)
    if bits == 8:
        out += flat.astype(np.int8).tobytes()
    else:
        v = flat.astype(np.int64)
        if v.size % 2:
            v = np.concatenate([v, np.zeros(1, dtype=np.int64)])
        nib = (v & 0xF).reshape(-1, 2)
        out += (nib[:, 0] | (nib[:, 1] << 4)).astype(np.uint8).tobytes()
    out += struct.pack("<I", zlib.crc32(bytes(out)) & 0xFFFFFFFF)
    return bytes(out)


# ---------------------------------------------------------------------------
# conv lowering (harness/layers.py:96-158)
# ---------------------------------------------------------------------------

def conv_out_hw(H: int, W: int, k: int, s: int, p: int):
    return (H + 2 * p - k) // s + 1, (W + 2 * p - k) // s + 1


def im2col(x: np.ndarray, k: int, s: int, p: int) -> np.ndarray:
    """(B, C, H, W) -> (B, Ho*Wo, C*k*k); column index c*k*k + i*k + j."""
    B, C, H, W = x.shape
    Ho, Wo = conv_out_hw(H, W, k, s, p)
    xp = np.pad(x, ((0, 0), (0, 0), (p, p), (p, p)))
    taps = np.stack([np.stack([xp[:, :, i:i + s * Ho:s, j:j + s * Wo:s] for j in range(k)], 2)
                     for i in range(k)], 2)          # (B, C, k, k, Ho, Wo)
    return np.ascontiguousarray(taps.transpose(0, 4, 5, 1, 2, 3)).reshape(B, Ho * Wo, C * k * k)


def col2im(cols: np.ndarray, x_shape, k: int, s: int, p: int) -> np.ndarray:
    """Scatter-add inverse of im2col, taps accumulated in (i, j) order in the
    column dtype (fp32 for the dequantized path, int64 for accumulators)."""
    B, C, H, W = x_shape
    Ho, Wo = conv_out_hw(H, W, k, s, p)
    c6 = cols.reshape(B, Ho, Wo, C, k, k)
    acc = np.zeros((B, C, H + 2 * p, W + 2 * p), dtype=cols.dtype)
    for i in range(k):
        for j in range(k):
            acc[:, :, i:i + s * Ho:s, j:j + s * Wo:s] += c6[..., i, j].transpose(0, 3, 1, 2)
    return np.ascontiguousarray(acc[:, :, p:p + H, p:p + W])


def conv2d_hlq_backward(x: np.ndarray, w4: np.ndarray, gy: np.ndarray, stride: int, pad: int,
                        rank: int = 8, bits_gx: int = 4, bits_gw: int = 8, n: int = 16,
                        extra: float | None = None, stages: dict | None = None):
    """Conv2d.forward's ACBP + Conv2d.backward (layers.py:141-158)."""
    O, C, k, _ = w4.shape
    B = x.shape[0]
    cols = im2col(x, k, stride, pad)
    gy3 = np.ascontiguousarray(gy.transpose(0, 2, 3, 1).reshape(B, -1, O))
    gcols, gw = hlq_backward(cols, w4.reshape(O, -1), gy3, rank, bits_gx, bits_gw, n,
                             extra=extra, stages=stages)
    gx = col2im(gcols, x.shape, k, stride, pad)
    return gx, gw.reshape(O, C, k, k)


# ---------------------------------------------------------------------------
# synthetic inputs
# ---------------------------------------------------------------------------

def make_inputs(seed: int, x_shape, w_shape, gy_shape):
    rng = np.random.default_rng(seed)
    x = rng.standard_normal(x_shape).astype(F32)
    fan_in = int(np.prod(w_shape[1:]))
    w = (rng.standard_normal(w_shape) * np.sqrt(2.0 / fan_in)).astype(F32)
    gy = (rng.lognormal(0.0, 1.4, size=gy_shape) * rng.choice([-1.0, 1.0], size=gy_shape)
          * 1e-3).astype(F32)
    return x, w, gy
