"""GPU ACBP container (reference acbp.py, test_acbp.py): pack bytes equal to the
reference's acbp_pack (golden fixtures), byte-exact round trips, and the
reference's validation rules (FormatError + byte offset)."""
import json
import os
import struct
import zlib

import numpy as np
import pytest
import torch

from oracle import hlq_oracle as orc

from .conftest import GOLDEN

pytestmark = pytest.mark.gpu

MANIFEST = json.load(open(os.path.join(GOLDEN, "MANIFEST.json")))
CONTAINERS = [c for c in MANIFEST["cases"] if c.startswith("acbp_")]


@pytest.fixture(scope="module")
def mods():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2406_15102_b200 as h
    from paper_2406_15102_b200 import acbp
    return h, acbp


def compress(h, x, bases, bits, pad_small=False):
    plan = h.HadamardPlan(block_size=16, basis_indices=tuple(int(b) for b in bases))
    return h.acbp_compress(torch.from_numpy(np.ascontiguousarray(x)).cuda(), plan, bits=bits,
                           pad_small_axes=pad_small)


@pytest.mark.parametrize("case", CONTAINERS)
def test_pack_matches_reference_bytes(mods, case):
    h, acbp = mods
    g = dict(np.load(os.path.join(GOLDEN, case + ".npz")))
    a = compress(h, g["x"], g["bases"], int(g["bits"]), bool(g["pad_small"]))
    buf = acbp.acbp_pack(a)
    assert acbp.to_bytes(buf) == g["container"].tobytes()
    back = acbp.acbp_unpack(acbp.from_bytes(g["container"].tobytes()))
    assert back.orig_shape == tuple(g["x"].shape) and back.axis == int(g["axis"])
    assert back.quantized.bits == int(g["bits"])
    assert float(back.quantized.scale.cpu()) == float(g["scale"])
    assert np.array_equal(back.reference_payload().cpu().numpy().reshape(-1), g["payload"].reshape(-1))
    assert acbp.to_bytes(acbp.acbp_pack(back)) == g["container"].tobytes()  # byte-exact round trip


def test_large_container_crc_and_round_trip(mods):
    """ViT-B/16 fc1 input size (10 MB payload): the parallel CRC over many 4 KiB
    chunks equals zlib's, and the payload survives the round trip."""
    h, acbp = mods
    torch.manual_seed(0)
    x = torch.randn(128, 197, 768, device="cuda", dtype=torch.bfloat16)
    a = h.acbp_compress(x, h.HadamardPlan())
    buf = acbp.acbp_pack(a)
    raw = acbp.to_bytes(buf)
    assert struct.unpack("<I", raw[-4:])[0] == zlib.crc32(raw[:-4]) & 0xFFFFFFFF
    assert len(raw) == acbp.header_nbytes() + a.payload_nbytes
    back = acbp.acbp_unpack(buf)
    assert torch.equal(back.quantized.payload[:, :back.k], a.quantized.payload[:, :a.k])
    ref = orc.acbp_container(a.reference_payload().cpu().numpy(), 8, 16, h.HadamardPlan().basis_indices,
                             128, 197, 768, a.quantized.scale.cpu().numpy()[0])
    assert raw == ref


def _buf(mods):
    h, acbp = mods
    rng = np.random.default_rng(0)
    x = rng.standard_normal((4, 32, 12)).astype(np.float32)
    return bytearray(acbp.to_bytes(acbp.acbp_pack(compress(h, x, tuple(range(8)), 8))))


def _unpack(mods, b):
    _, acbp = mods
    return acbp.acbp_unpack(acbp.from_bytes(bytes(b)))


def test_validation_offsets(mods):
    from paper_2406_15102_b200.errors import FormatError
    buf = _buf(mods)
    for pos, val, off in ((0, 0x00, 0), (4, 99, 4), (6, 5, 6), (7, 3, 7), (8, 0, 8), (12, 2, 12)):
        b = bytearray(buf)
        b[pos] = val
        with pytest.raises(FormatError) as e:
            _unpack(mods, b)
        assert e.value.offset == off
    with pytest.raises(FormatError):
        _unpack(mods, buf[:10])
    with pytest.raises(FormatError):
        _unpack(mods, buf[:-1])
    # crc catches payload corruption
    b = bytearray(buf)
    b[33 + 5] ^= 0x01
    with pytest.raises(FormatError) as e:
        _unpack(mods, b)
    assert e.value.offset == len(buf) - 4
    # out-of-range payload value with a repaired CRC: the range check fires first
    b = bytearray(buf)
    b[33 + 3] = 0x80
    b[-4:] = struct.pack("<I", zlib.crc32(bytes(b[:-4])) & 0xFFFFFFFF)
    with pytest.raises(FormatError) as e:
        _unpack(mods, b)
    assert e.value.offset == 33 + 3


def test_int4_padding_nibble(mods):
    from paper_2406_15102_b200.errors import FormatError
    h, acbp = mods
    g = dict(np.load(os.path.join(GOLDEN, "acbp_c4_odd.npz")))
    b = bytearray(g["container"].tobytes())
    b[-5] |= 0x10  # high nibble of the last payload byte (odd count)
    b[-4:] = struct.pack("<I", zlib.crc32(bytes(b[:-4])) & 0xFFFFFFFF)
    with pytest.raises(FormatError) as e:
        _unpack(mods, b)
    assert e.value.offset == len(b) - 5


def test_bit_flip_fuzz_always_format_error(mods):
    from paper_2406_15102_b200.errors import FormatError
    rng = np.random.default_rng(99)
    h, acbp = mods
    x = rng.standard_normal((2, 16, 5)).astype(np.float32)
    buf = acbp.to_bytes(acbp.acbp_pack(compress(h, x, tuple(range(8)), 8)))
    for _ in range(120):
        b = bytearray(buf)
        b[int(rng.integers(0, len(b)))] ^= 1 << int(rng.integers(0, 8))
        with pytest.raises(FormatError):
            _unpack(mods, b)
