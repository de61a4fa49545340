"""Torch-facing wrappers over the C-ABI stage primitives.

Every function takes / returns CUDA tensors, allocates outputs with the torch
caching allocator, and enqueues work on torch's current stream.  There is no
CPU path: a CPU tensor raises ParameterError and a missing library raises
HLQLibraryError.
"""
from __future__ import annotations

import ctypes
import os

import torch

from . import _lib
from .errors import DimensionError, ParameterError

QMAX = {4: 7, 8: 127}
STATS_WORDS = 128  # HLQ_STATS_WS_BYTES / 4

# ---------------------------------------------------------------------------
# launch accounting / tracing (bench.py's gpu_launches and roofline inputs)
# ---------------------------------------------------------------------------
LAUNCHES = [0]  # number of libhlq kernels enqueued by this process
_TRACE = [None]


class Trace:
    """Records a CUDA event pair around every libhlq call on the launching
    stream, with the call's algorithmic bytes (transforms) or ops (GEMMs)."""

    def __init__(self):
        self.records = []  # (kind, key, start_event, end_event, bytes, ops, launches)

    def summary(self, by: str = "kind"):
        """Aggregate per kind ("transform", "gemm", ...) or per key (kind plus
        the call's operation and shape, e.g. "transform:dual:25216x3072")."""
        torch.cuda.synchronize()
        out = {}
        for kind, key, s, e, nbytes, nops, nl in self.records:
            d = out.setdefault(kind if by == "kind" else key,
                               {"calls": 0, "us": 0.0, "bytes": 0, "ops": 0, "launches": 0})
            d["calls"] += 1
            d["us"] += s.elapsed_time(e) * 1e3
            d["bytes"] += nbytes
            d["ops"] += nops
            d["launches"] += nl
        return out


class trace:
    def __enter__(self):
        self.t = Trace()
        _TRACE[0] = self.t
        return self.t

    def __exit__(self, *exc):
        _TRACE[0] = None
        return False


def _traced(kind: str, nbytes: int, nops: int, launches: int, fn, key: str | None = None):
    LAUNCHES[0] += launches
    tr = _TRACE[0]
    if tr is None:
        return fn()
    s = torch.cuda.Event(enable_timing=True)
    e = torch.cuda.Event(enable_timing=True)
    s.record()
    r = fn()
    e.record()
    tr.records.append((kind, key or kind, s, e, nbytes, nops, launches))
    return r


def pad16(n: int) -> int:
    return (int(n) + 15) & ~15


def _stream():
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def _first_tensor(args, kwargs):
    for a in list(args) + list(kwargs.values()):
        if torch.is_tensor(a):
            return a
        if isinstance(a, (list, tuple)) and a and torch.is_tensor(a[0]):
            return a[0]
        if isinstance(a, dict) and torch.is_tensor(a.get("a")):
            return a["a"]
    return None


def on_device(fn):
    """Run an op with its operands' device current: libhlq launches into the
    current CUDA context on torch's current stream of the current device, so
    a tensor on cuda:1 while cuda:0 is current must switch first (the check
    costs one cudaGetDevice when the device already matches)."""
    import functools

    @functools.wraps(fn)
    def wrapped(*args, **kwargs):
        t = _first_tensor(args, kwargs)
        if t is not None and t.is_cuda and t.device.index != torch.cuda.current_device():
            with torch.cuda.device(t.device):
                return fn(*args, **kwargs)
        return fn(*args, **kwargs)
    return wrapped


def _p(t):
    return ctypes.c_void_p(0 if t is None else t.data_ptr())


def dtype_code(t: torch.Tensor) -> int:
    if t.dtype == torch.float32:
        return _lib.HLQ_F32
    if t.dtype == torch.bfloat16:
        return _lib.HLQ_BF16
    raise ParameterError(f"HLQ kernels take float32 or bfloat16 inputs, got {t.dtype}")


def _cuda(t: torch.Tensor, what: str) -> torch.Tensor:
    if not t.is_cuda:
        raise ParameterError(f"{what} must be a CUDA tensor (the HLQ path has no CPU fallback)")
    return t if t.is_contiguous() else t.contiguous()


def _check_bits(bits):
    if bits not in (4, 8):
        raise ParameterError(f"bits must be 4 or 8, got {bits}")


def new_stats(device) -> torch.Tensor:
    """4 x uint32 statistics scratch: {amax, ~minnz} for the gx and gw operands."""
    return torch.zeros(4, dtype=torch.int32, device=device)


def quant_ht_cols(src: torch.Tensor, bits: int, want_stats: bool = True):
    """Q_bits(block-FWHT of every row of a (rows, cols) matrix along cols).
    Returns (codes (rows, pad16(cols)) int8, scale (1,) fp32, amax_bits (1,) int32);
    want_stats=False: the statistics stay in a library slot (no memset launch)
    and amax_bits is None."""
    _check_bits(bits)
    src = _cuda(src, "src")
    rows, cols = src.shape
    ld = pad16(cols)
    codes = torch.empty((rows, ld), dtype=torch.int8, device=src.device)
    scale = torch.empty(1, dtype=torch.float32, device=src.device)
    stats = torch.empty(STATS_WORDS, dtype=torch.int32, device=src.device) if want_stats else None
    _traced("transform", rows * cols * src.element_size() + rows * ld, 0, 1,
            lambda: _lib.call("hlq_quantize_ht_cols", _p(src), dtype_code(src), rows, cols, cols,
                              bits, _p(stats), _p(codes), ld, _p(scale), _stream()))
    return codes, scale, None if stats is None else stats[0:1]


def packed_ld(cols: int) -> int:
    """Row stride (bytes) of packed int4 codes for `cols` columns: pad16(cols) / 2
    rounded up to 16 (TMA row strides are 16-byte multiples)."""
    return (pad16(cols) // 2 + 15) & ~15


def unpack_int4(packed: torch.Tensor, cols: int) -> torch.Tensor:
    """int8 codes (rows, cols) from packed int4 rows (two per byte, low nibble
    first).  Torch ops -- for parity checks / stage dumps, not the hot path."""
    p = packed.view(torch.uint8).to(torch.int16)
    lo, hi = p & 0xF, p >> 4
    out = torch.stack([lo, hi], dim=-1).reshape(packed.shape[0], -1)[:, :cols]
    return torch.where(out >= 8, out - 16, out).to(torch.int8)


def quant_dual(src: torch.Tensor, segs: int, rows: int, cols: int, bitmap: int, bits_gx: int,
               bits_gw: int, ld_src: int | None = None, seg_src: int | None = None, colsum: bool = False,
               pack_gx: bool = False, want_stats: bool = True):
    """Both gy operands from one read per pass: HT along cols (gx) and the
    rank-r projection along rows (gw).  Returns
    (gx_codes (segs*rows, pad16(cols)), gx_scale, gw_codes (cols, pad16(K)), K, gw_scale, stats)
    and, with colsum, a 7th item: the fp32 column sums of src (cols,) -- the
    bias gradient -- computed from the same tiles.  pack_gx (4-bit gx codes):
    gx_codes is (segs*rows, packed_ld(cols)) uint8, two codes per byte, low
    nibble first (hlq_quantize_dual_ex) -- the A operand of gemm_i8(a_packed=True).
    want_stats=False: the statistics stay in a library slot (no memset launch), stats is None."""
    _check_bits(bits_gx)
    _check_bits(bits_gw)
    if pack_gx and bits_gx != 4:
        raise ParameterError("packed gx codes are 4-bit")
    src = _cuda(src, "src")
    ld_src = cols if ld_src is None else ld_src
    seg_src = rows * ld_src if seg_src is None else seg_src
    k = proj_rows_k(segs, rows, bin(bitmap).count("1"))
    ldk = max(pad16(k), 16)
    dev = src.device
    if pack_gx:
        cgx = torch.empty((segs * rows, packed_ld(cols)), dtype=torch.uint8, device=dev)
    else:
        cgx = torch.empty((segs * rows, pad16(cols)), dtype=torch.int8, device=dev)
    cgw = torch.empty((cols, ldk), dtype=torch.int8, device=dev)
    scales = torch.empty(2, dtype=torch.float32, device=dev)
    stats = torch.empty(STATS_WORDS, dtype=torch.int32, device=dev) if want_stats else None
    nbytes = segs * rows * cols * src.element_size() + cgx.numel() + cols * k
    key = f"transform:dual:{segs * rows}x{cols}:{src.dtype}".replace("torch.", "")
    cs = torch.empty(cols, dtype=torch.float32, device=dev) if colsum else None
    wsb = int(_lib.load().hlq_quantize_dual_colsum_ws(segs, rows, cols, bitmap)) if colsum else 0
    ws = torch.empty(max(wsb, 4), dtype=torch.uint8, device=dev) if colsum else None
    _traced("transform", nbytes + (cols * 4 if colsum else 0), 0, 1,
            lambda: _lib.call("hlq_quantize_dual_ex", _p(src), dtype_code(src), segs, rows, cols, ld_src, seg_src,
                              bitmap, bits_gx, bits_gw, _p(stats), _p(cgx), cgx.stride(0), int(pack_gx), _p(cgw),
                              ldk, _p(scales), _p(scales[1:]), _p(cs), _p(ws), wsb, _stream()),
            key=key)
    if colsum:
        return cgx, scales[0:1], cgw, k, scales[1:2], stats, cs
    return cgx, scales[0:1], cgw, k, scales[1:2], stats


def transform_pass(src: torch.Tensor, segs: int, rows: int, cols: int, ld_src: int, seg_src: int,
                   do_gx: bool, do_gw: bool, bitmap: int, bits_gx: int, bits_gw: int, mode: int,
                   stats: torch.Tensor, dst_gx=None, dst_gw=None, scale_gx=None, scale_gw=None):
    """One STATS (mode 0) or QUANT (mode 1) pass of the general transform
    (hlq_transform_pass); stats is a 4-word int32 tensor (see new_stats)."""
    src = _cuda(src, "src")
    nbytes = segs * rows * cols * src.element_size()
    _traced("transform", nbytes, 0, 1,
            lambda: _lib.call("hlq_transform_pass", _p(src), dtype_code(src), segs, rows, cols, ld_src,
                              seg_src, int(do_gx), int(do_gw), bitmap, bits_gx, bits_gw, mode,
                              _p(stats), _p(dst_gx), 0 if dst_gx is None else dst_gx.stride(0),
                              _p(dst_gw), 0 if dst_gw is None else dst_gw.stride(0), _p(scale_gx),
                              _p(scale_gw), _stream()))


def proj_rows_k(segs: int, rows: int, rank: int) -> int:
    return segs * ((rows + 15) // 16) * rank


def quant_proj_rows(src: torch.Tensor, segs: int, rows: int, cols: int, bitmap: int, bits: int,
                    ld_src: int | None = None, seg_src: int | None = None, want_stats: bool = True):
    """Q_bits(rank-r block projection along rows), written transposed.
    Returns (codes (cols, pad16(K)) int8, K, scale (1,), amax_bits (1,));
    want_stats=False: library statistics slot, amax_bits None."""
    _check_bits(bits)
    src = _cuda(src, "src")
    ld_src = cols if ld_src is None else ld_src
    seg_src = rows * ld_src if seg_src is None else seg_src
    k = proj_rows_k(segs, rows, bin(bitmap).count("1"))
    ld = max(pad16(k), 16)
    codes = torch.empty((cols, ld), dtype=torch.int8, device=src.device)
    scale = torch.empty(1, dtype=torch.float32, device=src.device)
    stats = torch.empty(STATS_WORDS, dtype=torch.int32, device=src.device) if want_stats else None
    _traced("transform", segs * rows * cols * src.element_size() + cols * k, 0, 1,
            lambda: _lib.call("hlq_quantize_proj_rows", _p(src), dtype_code(src), segs, rows, cols,
                              ld_src, seg_src, bitmap, bits, _p(stats), _p(codes), ld, _p(scale),
                              _stream()),
            key=f"transform:proj:{segs * rows}x{cols}:{src.dtype}".replace("torch.", ""))
    return codes, k, scale, None if stats is None else stats[2:3]


def quant_weights(weights, bits: int, bf16: bool = False):
    """Q_bits(HT_O(W)) for a list of fp32 CUDA weights (O, I) in one launch.
    Returns [(codes (I, pad16(O)) int8, scale (1,) fp32)] -- the same as
    quant_proj_rows(W, 1, O, I, 0xFFFF, bits)[0, 2] per tensor -- or, with
    bf16, [(codes, scale, W as bf16 (O, I))] (the cast rides on the same read)."""
    _check_bits(bits)
    n = len(weights)
    if n == 0:
        return []
    if n > 128:
        out = []
        for i in range(0, n, 128):
            out += quant_weights(weights[i:i + 128], bits, bf16)
        return out
    dev = weights[0].device
    ws_ = [_cuda(w, "weight") for w in weights]
    for w in ws_:
        if w.dtype != torch.float32 or w.dim() != 2:
            raise ParameterError("batched weight codes take 2-D float32 weights")
    codes = [torch.empty((w.shape[1], pad16(w.shape[0])), dtype=torch.int8, device=dev) for w in ws_]
    wbf = [torch.empty(w.shape, dtype=torch.bfloat16, device=dev) for w in ws_] if bf16 else None
    scales = torch.empty(n, dtype=torch.float32, device=dev)
    wsb = int(_lib.load().hlq_quantize_weights_ws(n))
    scratch = torch.empty(wsb, dtype=torch.uint8, device=dev)
    P = ctypes.c_void_p * n
    I64 = ctypes.c_int64 * n
    wp = P(*[w.data_ptr() for w in ws_])
    cp = P(*[c.data_ptr() for c in codes])
    sp = P(*[scales.data_ptr() + 4 * i for i in range(n)])
    bp = P(*[b.data_ptr() for b in wbf]) if bf16 else None
    Os = I64(*[w.shape[0] for w in ws_])
    Is = I64(*[w.shape[1] for w in ws_])
    lds = I64(*[c.stride(0) for c in codes])
    nbytes = sum(w.numel() * 4 + c.numel() + (w.numel() * 2 if bf16 else 0) for w, c in zip(ws_, codes))
    _traced("transform", nbytes, 0, 1,
            lambda: _lib.call("hlq_quantize_weights_ex", n, wp, Os, Is, bits, cp, lds, sp, bp, _p(scratch), wsb,
                              _stream()),
            key=f"transform:weights:{n}")
    if bf16:
        return [(c, scales[i:i + 1], wbf[i]) for i, c in enumerate(codes)]
    return [(c, scales[i:i + 1]) for i, c in enumerate(codes)]


def quant_stochastic(src: torch.Tensor, segs: int, rows: int, cols: int, ld_src: int, seg_src: int,
                     along_cols: bool, bitmap: int, bits: int, seed: int, counter: int = 0,
                     index_kind: int = 1, l2: int = 0, o2: int = 0):
    """True stochastic rounding of the transformed source (hlq_quantize_stochastic).
    along_cols: HT along cols -> (codes (segs*rows, pad16(cols)), scale, stats);
    else the projection along rows -> (codes (cols, pad16(K)), scale, stats, K)."""
    _check_bits(bits)
    src = _cuda(src, "src")
    dev = src.device
    if along_cols:
        ld = pad16(cols)
        codes = torch.empty((segs * rows, ld), dtype=torch.int8, device=dev)
        k = None
    else:
        k = proj_rows_k(segs, rows, bin(bitmap).count("1"))
        ld = max(pad16(k), 16)
        codes = torch.empty((cols, ld), dtype=torch.int8, device=dev)
    scale = torch.empty(1, dtype=torch.float32, device=dev)
    stats = torch.empty(STATS_WORDS, dtype=torch.int32, device=dev)
    _traced("transform", segs * rows * cols * src.element_size() + codes.numel(), 0, 2,
            lambda: _lib.call("hlq_quantize_stochastic", _p(src), dtype_code(src), segs, rows, cols, ld_src,
                              seg_src, int(along_cols), bitmap, bits, int(seed), int(counter), index_kind, l2, o2,
                              _p(stats), _p(codes), ld, _p(scale), _stream()),
            key=f"transform:stochastic:{segs * rows}x{cols}")
    amax = stats[0:1] if along_cols else stats[2:3]
    if along_cols:
        return codes, scale, amax
    return codes, scale, amax, k


def basis_energy(src: torch.Tensor, segs: int, rows: int, cols: int, ld_src: int | None = None,
                 seg_src: int | None = None):
    """Per-basis sums of |coefficient| of the block transform along rows
    (hlq_basis_energy) -> (sums (16,) float64 tensor, number of blocks x columns)."""
    src = _cuda(src, "src")
    ld_src = cols if ld_src is None else ld_src
    seg_src = rows * ld_src if seg_src is None else seg_src
    energy = torch.empty(16, dtype=torch.float64, device=src.device)
    _traced("transform", segs * rows * cols * src.element_size(), 0, 1,
            lambda: _lib.call("hlq_basis_energy", _p(src), dtype_code(src), segs, rows, cols, ld_src, seg_src,
                              _p(energy), _stream()))
    return energy, segs * ((rows + 15) // 16) * cols


# ---------------------------------------------------------------------------
# baseline-strategy transforms (hlq_xform_*)
# ---------------------------------------------------------------------------

def _xview(src, segs, rows, cols, src_strides, bitmap, dst_strides, idx_strides=(0, 0, 0)):
    v = _lib.Xform()
    v.src = src.data_ptr()
    v.src_dtype = dtype_code(src) if src.dtype != torch.float32 else _lib.HLQ_F32
    v.segs, v.rows, v.cols = int(segs), int(rows), int(cols)
    v.bitmap = int(bitmap)
    for i in range(3):
        v.src_stride[i] = int(src_strides[i])
        v.dst_stride[i] = int(dst_strides[i])
        v.idx_stride[i] = int(idx_strides[i])
    return v


def xform_quantize(src: torch.Tensor, segs: int, rows: int, cols: int, src_strides, bitmap: int,
                   dst: torch.Tensor, dst_strides, bits: int, seed: int | None = None, counter: int = 0,
                   idx_strides=(0, 0, 0)):
    """Q_bits of the strided view's outputs into the int8 tensor dst (pseudo-
    stochastic rounding, or Philox draws when seed is given).  Returns
    (scale (1,) fp32, amax_bits (1,) int32)."""
    _check_bits(bits)
    src = _cuda(src, "src")
    if dst.dtype != torch.int8:
        raise ParameterError("codes must be int8")
    v = _xview(src, segs, rows, cols, src_strides, bitmap, dst_strides, idx_strides)
    scale = torch.empty(1, dtype=torch.float32, device=src.device)
    stats = torch.empty(STATS_WORDS, dtype=torch.int32, device=src.device)
    rounding = 0 if seed is None else 1
    _traced("transform", src.numel() * src.element_size() + dst.numel(), 0, 2,
            lambda: _lib.call("hlq_xform_quantize", ctypes.byref(v), bits, rounding, int(seed or 0),
                              int(counter), _p(stats), _p(dst), _p(scale), _stream()),
            key=f"transform:xform_quant:{segs * rows}x{cols}")
    return scale, stats[0:1]


def xform_project(src: torch.Tensor, segs: int, rows: int, cols: int, src_strides, bitmap: int,
                  dst: torch.Tensor, dst_strides) -> torch.Tensor:
    """The strided view's (transformed) outputs in float32 into dst."""
    src = _cuda(src, "src")
    if dst.dtype != torch.float32:
        raise ParameterError("projection output must be float32")
    v = _xview(src, segs, rows, cols, src_strides, bitmap, dst_strides)
    _traced("transform", src.numel() * src.element_size() + dst.numel() * 4, 0, 1,
            lambda: _lib.call("hlq_xform_project_f32", ctypes.byref(v), _p(dst), _stream()),
            key=f"transform:xform_f32:{segs * rows}x{cols}")
    return dst


def xform_unproject(coeffs: torch.Tensor, segs: int, rows: int, cols: int, src_strides, bitmap: int,
                    dst: torch.Tensor, dst_strides) -> torch.Tensor:
    """_unproject_axis: kept coefficients (s, k, c) -> float32 (s, r, c), r < rows."""
    coeffs = _cuda(coeffs, "coefficients")
    if coeffs.dtype != torch.float32 or dst.dtype != torch.float32:
        raise ParameterError("unprojection runs in float32")
    v = _xview(coeffs, segs, rows, cols, src_strides, bitmap, dst_strides)
    _traced("transform", coeffs.numel() * 4 + dst.numel() * 4, 0, 1,
            lambda: _lib.call("hlq_xform_unproject_f32", ctypes.byref(v), _p(dst), _stream()),
            key=f"transform:unproject:{segs * rows}x{cols}")
    return dst


def proj_rows_amax(src: torch.Tensor, segs: int, rows: int, cols: int, bitmap: int,
                   stats: torch.Tensor, ld_src: int | None = None, seg_src: int | None = None):
    """Accumulate the transformed statistics (IEEE bits, atomic max) into stats[2:4]
    (`stats` from new_stats(); all-reduce(MAX) it across ranks for global scales)."""
    src = _cuda(src, "src")
    ld_src = cols if ld_src is None else ld_src
    seg_src = rows * ld_src if seg_src is None else seg_src
    _lib.call("hlq_proj_rows_amax", _p(src), dtype_code(src), segs, rows, cols, ld_src, seg_src,
              bitmap, _p(stats), _stream())


def proj_rows_quant(src: torch.Tensor, segs: int, rows: int, cols: int, bitmap: int, bits: int,
                    stats: torch.Tensor, ld_src: int | None = None, seg_src: int | None = None):
    src = _cuda(src, "src")
    ld_src = cols if ld_src is None else ld_src
    seg_src = rows * ld_src if seg_src is None else seg_src
    k = proj_rows_k(segs, rows, bin(bitmap).count("1"))
    ld = max(pad16(k), 16)
    codes = torch.empty((cols, ld), dtype=torch.int8, device=src.device)
    scale = torch.empty(1, dtype=torch.float32, device=src.device)
    _lib.call("hlq_proj_rows_quant", _p(src), dtype_code(src), segs, rows, cols, ld_src, seg_src,
              bitmap, bits, _p(stats), _p(codes), ld, _p(scale), _stream())
    return codes, k, scale


def gemm_i8(a: torch.Tensor, b: torch.Tensor, m: int, n: int, k: int, bits_a: int, bits_b: int,
            sa: torch.Tensor, sb: torch.Tensor, extra: float = 1.0, exact: bool = True,
            out_dtype=torch.float32, want_acc: bool = False, want_out: bool = True,
            groups: int = 1, a_gstride: int | None = None, b_gstride: int | None = None,
            a_packed: bool = False):
    """D[m, n] = sum_(g,k) A[g][m, k] B[g][n, k] on K-major int8 codes, fused dequant.
    Returns (out or None, acc or None)."""
    if a_packed:
        return _gemm_i4a(a, b, m, n, k, bits_b, sa, sb, extra, exact, out_dtype)
    if a.dtype != torch.int8 or b.dtype != torch.int8:
        raise ParameterError("GEMM operands must be int8 codes")
    dev = a.device
    out = torch.empty((m, n), dtype=out_dtype, device=dev) if want_out else None
    acc = torch.empty((m, n), dtype=torch.int32, device=dev) if want_acc else None
    lda, ldb = a.stride(0), b.stride(0)
    a_gs = lda * m if a_gstride is None else a_gstride
    b_gs = ldb * n if b_gstride is None else b_gstride
    # split-K workspace (the dW products: few output tiles, long K); stream-ordered
    # caching-allocator memory, no initialisation needed
    wsb = int(_lib.load().hlq_gemm_i8_ws_bits(m, n, k, groups, bits_a, bits_b)) if m > 0 and n > 0 else 0
    ws = torch.empty(wsb, dtype=torch.uint8, device=dev) if wsb else None
    _traced("gemm", 0, 2 * m * n * k * groups, 1,
            lambda: _lib.call("hlq_gemm_i8_ex", _p(a), lda, a_gs, _p(b), ldb, b_gs, m, n, k,
                              groups, bits_a, bits_b, _p(sa), _p(sb), float(extra),
                              _lib.HLQ_EPI_EXACT if exact else _lib.HLQ_EPI_FAST, _p(out),
                              _lib.HLQ_BF16 if out_dtype == torch.bfloat16 else _lib.HLQ_F32, n,
                              _p(acc), n, _p(ws), wsb, _stream()),
            key=f"gemm:{m}x{n}x{k * groups}")
    return out, acc


def _gemm_i4a(a, b, m, n, k, bits_b, sa, sb, extra, exact, out_dtype):
    """gemm_i8 with A as packed int4 codes (uint8 (m, >= ceil(k/2)), low nibble
    first): hlq_gemm_i4a_ex sign-extends them to int8 in shared memory."""
    if a.dtype != torch.uint8 or b.dtype != torch.int8:
        raise ParameterError("packed GEMM: A uint8 (two int4 codes per byte), B int8 codes")
    out = torch.empty((m, n), dtype=out_dtype, device=a.device)
    _traced("gemm", 0, 2 * m * n * k, 1,
            lambda: _lib.call("hlq_gemm_i4a_ex", _p(a), a.stride(0), a.stride(0) * m, _p(b), b.stride(0),
                              b.stride(0) * n, m, n, k, 1, bits_b, _p(sa), _p(sb), float(extra),
                              _lib.HLQ_EPI_EXACT if exact else _lib.HLQ_EPI_FAST, _p(out),
                              _lib.HLQ_BF16 if out_dtype == torch.bfloat16 else _lib.HLQ_F32, n, None, 0,
                              _stream()),
            key=f"gemm:i4a:{m}x{n}x{k}")
    return out, None


# >= 16 K blocks of 128 bytes in BOTH products (hlq_gemm.cu gemm_i8_pair2_eligible;
# HLQ_GEMM_PAIR_MINK overrides both sides for A/B measurements)
PAIR_MIN_K = int(os.environ.get("HLQ_GEMM_PAIR_MINK", "16")) * 128


def pair_eligible(m0: int, m1: int, k0: int, k1: int, n0: int = 0, n1: int = 0) -> bool:
    """True when hlq_gemm_i8_multi runs two products as ONE CTA-pair launch
    (mirror of hlq_gemm.cu gemm_i8_pair2_eligible): both >= 256 rows, each
    contraction long (>= 16 K blocks) or its output wide (N >= 2048, e.g. the
    ViT fc2 dX).  Otherwise the caller issues two gemm_i8 calls, which keeps the
    split-K planner for short-M products (the multi entry's sequential fallback
    runs without a split-K workspace).  HLQ_PAIR=0 disables the fused launch
    (A/B measurements)."""
    if os.environ.get("HLQ_PAIR", "1") == "0":
        return False
    for k, n in ((k0, n0), (k1, n1)):
        nk = (k + 127) // 128
        if not (k > PAIR_MIN_K - 128 or (n >= 2048 and nk >= 2)):
            return False
    # (contractions past the int32-exact bound run as K chunks through gemm_i8)
    return max(k0, k1) * 127 * 127 < 2 ** 31 and min(m0, m1) >= 256


def gemm_i8_pair(p0: dict, p1: dict):
    """Two independent products (typically a layer's dX and dW) in one call:
    each dict holds gemm_i8's arguments (a, b, m, n, k, bits_a, bits_b, sa, sb,
    extra, out_dtype; fast epilogue, single K group).  With long contractions
    they run as one CTA-pair launch over both products' tiles
    (hlq_gemm_i8_multi).  Returns (out0, out1)."""
    outs, descs = [], []
    for q in (p0, p1):
        a, b = q["a"], q["b"]
        packed = bool(q.get("a_packed", False))
        if a.dtype != (torch.uint8 if packed else torch.int8) or b.dtype != torch.int8:
            raise ParameterError("GEMM operands must be int8 codes (A: uint8 packed int4 with a_packed)")
        m, n, k = q["m"], q["n"], q["k"]
        od = q.get("out_dtype", torch.float32)
        out = torch.empty((m, n), dtype=od, device=a.device)
        outs.append(out)
        descs.append(_lib.GemmDesc(a.data_ptr(), a.stride(0), a.stride(0) * m, b.data_ptr(), b.stride(0),
                                   b.stride(0) * n, m, n, k, 1, q["bits_a"], q["bits_b"], q["sa"].data_ptr(),
                                   q["sb"].data_ptr(), float(q.get("extra", 1.0)), _lib.HLQ_EPI_FAST,
                                   out.data_ptr(), _lib.HLQ_BF16 if od == torch.bfloat16 else _lib.HLQ_F32, n, None,
                                   0, int(packed)))
    arr = (_lib.GemmDesc * 2)(*descs)
    ops_ = 2 * sum(q["m"] * q["n"] * q["k"] for q in (p0, p1))
    _traced("gemm", 0, ops_, 1, lambda: _lib.call("hlq_gemm_i8_multi", 2, ctypes.cast(arr, ctypes.c_void_p),
                                                  _stream()),
            key=f"gemm:pair:{p0['m']}x{p0['n']}x{p0['k']}+{p1['m']}x{p1['n']}x{p1['k']}")
    return outs[0], outs[1]


def conv_out_hw(H: int, W: int, k: int, stride: int, pad: int):
    return (H + 2 * pad - k) // stride + 1, (W + 2 * pad - k) // stride + 1


def conv_acbp(x_nhwc: torch.Tensor, k: int, stride: int, pad: int, bitmap: int, bits: int, want_stats: bool = True):
    """ACBP of im2col(x) along the output-pixel axis, from channels-last x
    (B, H, W, C) viewed as a contiguous tensor.  Returns (codes (C*k*k, pad16(K)), K, scale, amax)."""
    _check_bits(bits)
    x_nhwc = _cuda(x_nhwc, "x")
    B, H, W, C = x_nhwc.shape
    Ho, Wo = conv_out_hw(H, W, k, stride, pad)
    kk = B * ((Ho * Wo + 15) // 16) * bin(bitmap).count("1")
    ld = max(pad16(kk), 16)
    codes = torch.empty((C * k * k, ld), dtype=torch.int8, device=x_nhwc.device)
    scale = torch.empty(1, dtype=torch.float32, device=x_nhwc.device)
    stats = torch.empty(STATS_WORDS, dtype=torch.int32, device=x_nhwc.device) if want_stats else None
    nbytes = x_nhwc.numel() * x_nhwc.element_size() + C * k * k * kk
    _traced("transform", nbytes, 0, 2,
            lambda: _lib.call("hlq_conv_acbp_compress", _p(x_nhwc), dtype_code(x_nhwc), B, H, W, C, k,
                              stride, pad, bitmap, bits, _p(codes), ld, _p(scale), _p(stats),
                              _stream()),
            key=f"transform:conv_acbp:{B}x{H}x{W}x{C}:k{k}s{stride}")
    return codes, kk, scale, None if stats is None else stats[2:3]


def conv_acbp_pass(x_nhwc: torch.Tensor, k: int, stride: int, pad: int, bitmap: int, bits: int, mode: int,
                   stats: torch.Tensor, codes: torch.Tensor | None = None, scale: torch.Tensor | None = None):
    """One pass of the conv ACBP (hlq_conv_acbp_pass): mode 0 accumulates the
    statistics into stats[2:4], mode 1 writes the codes with the scale they imply."""
    x_nhwc = _cuda(x_nhwc, "x")
    B, H, W, C = x_nhwc.shape
    _lib.call("hlq_conv_acbp_pass", _p(x_nhwc), dtype_code(x_nhwc), B, H, W, C, k, stride, pad, bitmap, bits, mode,
              _p(stats), _p(codes), 0 if codes is None else codes.stride(0), _p(scale), _stream())
    LAUNCHES[0] += 1


def conv_dgrad_i8(gcodes: torch.Tensor, B: int, Ho: int, Wo: int, O: int, wcodes: torch.Tensor, C: int,
                  k: int, pad: int, bits: int, sg: torch.Tensor, sw: torch.Tensor, exact: bool = False,
                  out_dtype=torch.bfloat16, want_acc: bool = False, stride: int = 1, H: int | None = None,
                  W: int | None = None):
    """Implicit-GEMM dX (B, H, W, C) channels-last from the gx codes
    (B*Ho*Wo, >= O) and the W codes (C*k*k, >= O) -- no dcols tensor, no
    col2im; stride > 1 runs as stride^2 output phases (hlq_conv_dgrad_i8_ex).
    H / W: the forward input extent (default: the stride-1 one).  Returns (dx, acc or None)."""
    if H is None:
        H = (Ho - 1) * stride + k - 2 * pad
    if W is None:
        W = (Wo - 1) * stride + k - 2 * pad
    dx = torch.empty((B, H, W, C), dtype=out_dtype, device=gcodes.device)
    acc = torch.empty((B * H * W, C), dtype=torch.int32, device=gcodes.device) if want_acc else None
    _traced("gemm", 0, 2 * B * Ho * Wo * C * k * k * pad16(O), 1 if stride == 1 else stride * stride,
            lambda: _lib.call("hlq_conv_dgrad_i8_ex", _p(gcodes), gcodes.stride(0), B, Ho, Wo, O, _p(wcodes),
                              wcodes.stride(0), C, k, stride, pad, H, W, bits, _p(sg), _p(sw),
                              _lib.HLQ_EPI_EXACT if exact else _lib.HLQ_EPI_FAST, _p(dx),
                              _lib.HLQ_BF16 if out_dtype == torch.bfloat16 else _lib.HLQ_F32, _p(acc),
                              _stream()),
            key=f"gemm:conv_dgrad:{B}x{Ho}x{Wo}x{O}->{C}:k{k}s{stride}")
    return dx, acc


def col2im(dcols: torch.Tensor, B: int, H: int, W: int, C: int, k: int, stride: int, pad: int,
           out_dtype=torch.float32, tap_major: bool = False) -> torch.Tensor:
    """dX (B, H, W, C) contiguous (= channels-last NCHW) from dcols (B*L, C*k*k)."""
    dcols = _cuda(dcols, "dcols")
    dx = torch.empty((B, H, W, C), dtype=out_dtype, device=dcols.device)
    _traced("col2im", dcols.numel() * dcols.element_size() + dx.numel() * dx.element_size(), 0, 1,
            lambda: _lib.call("hlq_col2im_ex", _p(dcols), dtype_code(dcols), dcols.stride(0), B, H, W, C,
                              k, stride, pad, 1 if tap_major else 0, _p(dx),
                              _lib.HLQ_BF16 if out_dtype == torch.bfloat16 else _lib.HLQ_F32,
                              _stream()))
    return dx


def amax_to_float(amax_bits: torch.Tensor) -> torch.Tensor:
    return amax_bits.view(torch.float32)


def check_finite(*amax_bits: torch.Tensor) -> None:
    """Raise ValueError (quantize.py:138-139) if a transformed operand held NaN/Inf.
    Synchronizes; used by the reference-mirroring API, not by the training path."""
    for a in amax_bits:
        for v in a.reshape(-1).tolist():
            if int(v) & 0xFFFFFFFF >= 0x7F800000:
                raise ValueError("cannot quantize non-finite values")


def require_dims(cond: bool, msg: str):
    if not cond:
        raise DimensionError(msg)


for _name in ("quant_ht_cols", "quant_dual", "transform_pass", "quant_proj_rows", "quant_weights",
              "quant_stochastic", "basis_energy", "xform_quantize", "xform_project", "xform_unproject",
              "proj_rows_amax", "proj_rows_quant", "gemm_i8", "gemm_i8_pair", "conv_acbp", "conv_acbp_pass",
              "conv_dgrad_i8",
              "col2im"):
    globals()[_name] = on_device(globals()[_name])
del _name
