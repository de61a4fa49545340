"""ACBP container on the GPU -- mirror of the reference's acbp.py (3-212).

    acbp_pack(acbp) -> uint8 CUDA tensor   (the container bytes, byte-exact
                                            with the reference's acbp_pack)
    acbp_unpack(buf) -> ACBPActivation     (validates like the reference:
                                            FormatError with the byte offset)
    header_nbytes()                        (container overhead)

The container is built and checked by libhlq_b200 kernels (payload transpose
from our K-major layout to the reference's C order, int4 nibble packing,
parallel CRC32); only the 33 header bytes visit the host on unpack.
``to_bytes`` / ``from_bytes`` move a container between host bytes (what the
reference's functions exchange) and the device.
"""
from __future__ import annotations

import ctypes

import torch

from . import _lib, ops
from .backprop import ACBPActivation, QuantizedTensor
from .errors import ParameterError
from .hadamard import HadamardPlan


def header_nbytes(ndims: int = 3, num_scales: int = 1) -> int:
    """acbp.py:210-212: header + scales + CRC."""
    return 13 + 4 * ndims + 4 + 4 * num_scales + 4


def acbp_pack(acbp: ACBPActivation) -> torch.Tensor:
    q = acbp.quantized
    plan = acbp.plan
    if plan.block_size > 16:
        raise ParameterError("container format supports block sizes up to 16")
    if getattr(q, "per_axis", None) is not None:
        raise ParameterError("container format supports per-tensor scales only")
    if len(acbp.orig_shape) != 3:
        raise ParameterError(f"expected an original shape (B, L, I), got {acbp.orig_shape}")
    B, L, I = acbp.orig_shape
    payload = q.payload
    rows, k = payload.shape[0], acbp.k
    lib = _lib.load()
    total = int(lib.hlq_acbp_container_bytes(rows, k, q.bits))
    dev = payload.device
    out = torch.empty(total, dtype=torch.uint8, device=dev)
    wsb = int(lib.hlq_acbp_ws(total))
    ws = torch.empty(wsb, dtype=torch.uint8, device=dev)
    scale = q.scale.reshape(1).to(torch.float32)
    with torch.cuda.device(dev):
        _lib.call("hlq_acbp_pack", ops._p(payload), payload.stride(0) if payload.dim() == 2 else max(k, 1), rows,
                  k, q.bits, plan.block_size, plan.basis_bitmap(), B, L, I, ops._p(scale), ops._p(out), total,
                  ops._p(ws), wsb, ops._stream())
    return out


def acbp_unpack(buf: torch.Tensor) -> ACBPActivation:
    if not isinstance(buf, torch.Tensor) or buf.dtype != torch.uint8 or not buf.is_cuda:
        raise ParameterError("acbp_unpack takes the container as a uint8 CUDA tensor (see from_bytes)")
    buf = buf.contiguous()
    n = buf.numel()
    info = _lib.AcbpInfo()
    _lib.call("hlq_acbp_parse", ops._p(buf), n, ctypes.byref(info), ops._stream())
    dev = buf.device
    ld = max(ops.pad16(info.K), 16)
    # int8: the unpack transpose writes every byte (padding columns zeroed); int4 leaves them
    alloc = torch.empty if info.bits == 8 else torch.zeros
    payload = alloc((info.rows, ld), dtype=torch.int8, device=dev)
    scale = torch.empty(1, dtype=torch.float32, device=dev)
    wsb = int(_lib.load().hlq_acbp_ws(n))
    ws = torch.empty(wsb, dtype=torch.uint8, device=dev)
    _lib.call("hlq_acbp_unpack", ops._p(buf), n, ctypes.byref(info), ops._p(payload), ld, ops._p(scale),
              ops._p(ws), wsb, ops._stream())
    plan = HadamardPlan.from_bitmap(info.block, info.bitmap)
    qt = QuantizedTensor(payload=payload, bits=info.bits, scale=scale)
    return ACBPActivation(quantized=qt, orig_shape=(int(info.B), int(info.L), int(info.I)), axis=int(info.axis),
                          plan=plan, k=int(info.K))


acbp_unpack = ops.on_device(acbp_unpack)


def to_bytes(buf: torch.Tensor) -> bytes:
    return bytes(buf.cpu().numpy().tobytes())


def from_bytes(data: bytes, device="cuda") -> torch.Tensor:
    return torch.frombuffer(bytearray(data), dtype=torch.uint8).to(device)
