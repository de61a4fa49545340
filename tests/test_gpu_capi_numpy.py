"""The C-ABI boundary exactly as the reference would bind it:
host numpy arrays in, numpy arrays out, device memory through the CUDA
runtime via ctypes -- no torch, no package code on the call path.

Entry points exercised, replacing the reference's Python functions:
  hlq_acbp_compress  <- acbp_compress    (backprop.py:373)
  hlq_grad_weight    <- hlq_grad_weight  (backprop.py:388)
  hlq_hq_grad_input  <- hq_grad_input    (backprop.py:350)
against the golden lin* fixtures produced by the reference itself, bit for
bit (exact fp64 dequant epilogue, extra = 1/B as the reference applies it).
"""
import ctypes
import ctypes.util
import json
import os

import numpy as np
import pytest

from .conftest import GOLDEN

pytestmark = pytest.mark.gpu

LIB = os.path.join(os.path.dirname(GOLDEN), "..", "paper_2406_15102_b200", "libhlq_b200.so")
MANIFEST = json.load(open(os.path.join(GOLDEN, "MANIFEST.json")))
LINEAR = [c for c in MANIFEST["cases"] if c.startswith("lin")]
_P, _I64, _I, _SZ, _D, _U32 = (ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_size_t, ctypes.c_double,
                               ctypes.c_uint32)
H2D, D2H = 1, 2


def _cudart():
    cands = [ctypes.util.find_library("cudart"), "libcudart.so", "libcudart.so.12",
             "/usr/local/cuda/lib64/libcudart.so"]
    try:  # the CUDA runtime torch ships (nvidia-cuda-runtime wheel), if present
        import nvidia.cuda_runtime as ncr
        d = os.path.join(list(ncr.__path__)[0], "lib")
        cands += [os.path.join(d, f) for f in sorted(os.listdir(d)) if f.startswith("libcudart.so")]
    except Exception:  # noqa: BLE001
        pass
    for c in cands:
        if not c:
            continue
        try:
            return ctypes.CDLL(c)
        except OSError:
            continue
    pytest.skip("no CUDA runtime library to bind")


class Binding:
    """What a maintainer would add to the reference as hlq/_b200.py."""

    ERR = {1: "DimensionError", 2: "ParameterError", 3: "StateError", 4: "ValueError"}

    def __init__(self):
        self.lib = ctypes.CDLL(os.path.abspath(LIB))
        self.rt = _cudart()
        L = self.lib
        L.hlq_last_error.restype = ctypes.c_char_p
        L.hlq_acbp_k.restype = _I64
        L.hlq_acbp_k.argtypes = [_I64, _I64, _I, _I]
        L.hlq_acbp_rows.restype = _I64
        L.hlq_acbp_rows.argtypes = [_I64, _I64, _I]
        L.hlq_acbp_compress.argtypes = [_P, _I, _I64, _I64, _I64, _I, _U32, _I, _P, _I64, _P, _P, _P]
        L.hlq_hq_grad_input_ws.restype = _SZ
        L.hlq_hq_grad_input_ws.argtypes = [_I64, _I64, _I64]
        L.hlq_hq_grad_input.argtypes = [_P, _I, _I64, _I64, _P, _I64, _I, _P, _I, _I, _P, _SZ, _P]
        L.hlq_grad_weight_ws.restype = _SZ
        L.hlq_grad_weight_ws.argtypes = [_I64, _I64, _I64, _I, _I]
        L.hlq_grad_weight.argtypes = [_P, _I64, _P, _P, _I, _I64, _I64, _I64, _I64, _I, _U32, _I, _D, _P, _I, _I,
                                      _P, _SZ, _P]
        self.rt.cudaMalloc.argtypes = [ctypes.POINTER(_P), _SZ]
        self.rt.cudaMemcpy.argtypes = [_P, _P, _SZ, _I]
        self.rt.cudaMemset.argtypes = [_P, _I, _SZ]
        self.rt.cudaFree.argtypes = [_P]
        self.live = []

    def check(self, st):
        if st:
            raise RuntimeError(f"{self.ERR.get(st, 'HLQLibraryError')}: {self.lib.hlq_last_error().decode()}")

    def dev(self, nbytes):
        p = _P()
        assert self.rt.cudaMalloc(ctypes.byref(p), max(int(nbytes), 16)) == 0
        self.rt.cudaMemset(p, 0, max(int(nbytes), 16))
        self.live.append(p)
        return p

    def put(self, a):
        a = np.ascontiguousarray(a)
        p = self.dev(a.nbytes)
        assert self.rt.cudaMemcpy(p, a.ctypes.data, a.nbytes, H2D) == 0
        return p

    def get(self, p, shape, dtype):
        out = np.empty(shape, dtype)
        assert self.rt.cudaMemcpy(out.ctypes.data, p, out.nbytes, D2H) == 0  # synchronising copy
        return out

    def free(self):
        for p in self.live:
            self.rt.cudaFree(p)
        self.live = []

    # --- the reference's functions, numpy in / numpy out -------------------
    def acbp_compress(self, x, bitmap, bits, axis):
        B, L, I = x.shape
        rank = bin(bitmap).count("1")
        k = self.lib.hlq_acbp_k(B, L, axis, rank)
        rows = self.lib.hlq_acbp_rows(L, I, axis)
        ld = max((k + 15) // 16 * 16, 16)
        d_x, d_pay, d_s, d_st = self.put(x.astype(np.float32)), self.dev(rows * ld), self.dev(4), self.dev(512)  # HLQ_STATS_WS_BYTES
        self.check(self.lib.hlq_acbp_compress(d_x, 0, B, L, I, axis, bitmap, bits, d_pay, ld, d_s, d_st, None))
        return (d_pay, ld, d_s), self.get(d_pay, (rows, ld), np.int8)[:, :k], self.get(d_s, (1,), np.float32)[0], k

    def hlq_grad_weight(self, acbp, gy, bitmap, bits, axis, I):
        d_pay, ld, d_s = acbp
        B, L, O = gy.shape
        ws = self.lib.hlq_grad_weight_ws(B, L, O, axis, bin(bitmap).count("1"))
        d_g, d_w, d_ws = self.put(gy.astype(np.float32)), self.dev(O * I * 4), self.dev(ws)
        self.check(self.lib.hlq_grad_weight(d_pay, ld, d_s, d_g, 0, B, L, O, I, axis, bitmap, bits, 1.0 / B, d_w,
                                            0, 0, d_ws, ws, None))
        return self.get(d_w, (O, I), np.float32)

    def hq_grad_input(self, gy, w, bits):
        B, L, O = gy.shape
        I = w.shape[1]
        T = B * L
        ws = self.lib.hlq_hq_grad_input_ws(T, O, I)
        d_g, d_w, d_x, d_ws = self.put(gy.astype(np.float32)), self.put(w.astype(np.float32)), self.dev(T * I * 4), \
            self.dev(ws)
        self.check(self.lib.hlq_hq_grad_input(d_g, 0, T, O, d_w, I, bits, d_x, 0, 0, d_ws, ws, None))
        return self.get(d_x, (B, L, I), np.float32)


@pytest.fixture(scope="module")
def binding():
    try:
        import torch
        if not torch.cuda.is_available():
            pytest.skip("no CUDA device")
    except ImportError:
        pass
    b = Binding()
    yield b
    b.free()


@pytest.mark.parametrize("case", LINEAR)
def test_reference_binding_bit_exact(binding, case):
    g = dict(np.load(os.path.join(GOLDEN, case + ".npz")))
    x, w, gy = g["x"], g["w"], g["gy"]
    bitmap = int(sum(1 << int(b) for b in g["bases"]))
    axis = int(g["axis"])
    bits_gx, bits_gw = int(g["bits_gx"]), int(g["bits_gw"])
    B, L, I = x.shape
    acbp, payload, sx, k = binding.acbp_compress(x, bitmap, bits_gw, axis)
    # payload is K-major: (I, K) for the token axis, (L*I, K) for the batch axis
    ref = g["x_codes"]
    if axis == 1:
        assert np.array_equal(payload.T, ref)
    else:
        # rows (l, i), column kb  ->  the reference's (K_b, L, I) flattened to rows kb*L + l
        assert np.array_equal(payload.reshape(L, I, k).transpose(2, 0, 1).reshape(-1, I), ref)
    assert np.float32(sx).tobytes() == np.float32(g["x_scale"]).tobytes()
    gw = binding.hlq_grad_weight(acbp, gy, bitmap, bits_gw, axis, I)
    gx = binding.hq_grad_input(gy, w, bits_gx)
    assert np.array_equal(gw, g["gw"]), "dW not bit-exact"
    assert np.array_equal(gx, g["gx"]), "dX not bit-exact"
