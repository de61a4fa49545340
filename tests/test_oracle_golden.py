"""Pin the CPU oracle (oracle/hlq_oracle.py) to the reference's own outputs.

The fixtures under tests/golden/ were produced by running the reference
(tests/golden/make_golden.py); every comparison here is bit-exact.
"""
import json
import os

import numpy as np
import pytest

from oracle import hlq_oracle as orc

from .conftest import GOLDEN

MANIFEST = json.load(open(os.path.join(GOLDEN, "MANIFEST.json")))
LINEAR = [c for c in MANIFEST["cases"] if c.startswith("lin")]
CONV = [c for c in MANIFEST["cases"] if c.startswith("conv")]


def load(name):
    return dict(np.load(os.path.join(GOLDEN, name + ".npz")))


def test_default_bases_match_reference():
    ref = json.load(open(os.path.join(GOLDEN, "bases16.json")))
    for r, idx in ref.items():
        assert list(orc.lowest_sequency_bases(16, int(r))) == idx
    assert orc.lowest_sequency_bases(16, 8) == (0, 2, 4, 6, 8, 10, 12, 14)
    assert orc.lowest_sequency_bases(16, 2) == (0, 8)


@pytest.mark.parametrize("case", LINEAR)
def test_linear_case_bit_exact(case):
    g = load(case)
    st = {}
    gx, gw = orc.hlq_backward(g["x"], g["w"], g["gy"], bases=tuple(g["bases"]),
                              bits_gx=int(g["bits_gx"]), bits_gw=int(g["bits_gw"]),
                              pad_small_axes=bool(g["pad_small"]), stages=st)
    for key in ("gx_codes_g", "gx_codes_w", "gx_acc", "x_codes", "gw_codes_g", "gw_acc"):
        assert np.array_equal(st[key], g[key]), key
    for key in ("gx_scale_g", "gx_scale_w", "x_scale", "gw_scale_g"):
        assert np.float32(st[key]).tobytes() == np.float32(g[key]).tobytes(), key
    assert st["axis"] == int(g["axis"])
    assert np.array_equal(gx, g["gx"])
    assert np.array_equal(gw, g["gw"])


@pytest.mark.parametrize("case", CONV)
def test_conv_case_bit_exact(case):
    g = load(case)
    st = {}
    gx, gw = orc.conv2d_hlq_backward(g["x"], g["w"], g["gy"], int(g["stride"]), int(g["pad"]),
                                     rank=int(g["rank"]), stages=st)
    for key in ("gx_codes_g", "gx_codes_w", "gx_acc", "x_codes", "gw_codes_g", "gw_acc"):
        assert np.array_equal(st[key], g[key]), key
    assert np.array_equal(gx, g["gx"])
    assert np.array_equal(gw, g["gw"])


def test_known_answers():
    c = load("ka_constant")
    codes, scale, axis = orc.acbp_compress(c["x"], orc.lowest_sequency_bases(16, 8))
    assert np.array_equal(codes, c["x_codes"]) and scale == c["x_scale"] == 1.0
    assert np.all(codes.reshape(2, 8, 3)[:, 0] == 127) and np.all(codes.reshape(2, 8, 3)[:, 1:] == 0)
    z = load("ka_zero")
    codes, scale, _ = orc.acbp_compress(z["x"], orc.lowest_sequency_bases(16, 8))
    assert scale == 1.0 and not codes.any()
    q = load("ka_quant")
    c4, s4 = orc.quantize(q["lattice"], 4)
    assert np.array_equal(c4, q["lattice_codes"]) and s4 == q["lattice_scale"]
    for bits in (4, 8):
        cb, sb = orc.quantize(q["ln"], bits)
        assert np.array_equal(cb, q[f"ln_codes{bits}"]) and sb == q[f"ln_scale{bits}"]


def test_fwht_stage_order_matters():
    """Reversing the stage order changes fp32 results: the order is part of the contract."""
    rng = np.random.default_rng(0)
    v = (rng.standard_normal((4096, 16)) * 1e3).astype(np.float32)
    fwd = orc.fwht_blocks(v)
    x = v.copy()
    for h in (8, 4, 2, 1):
        lo = np.array([i for i in range(16) if not i & h])
        a, b = x[:, lo], x[:, lo + h]
        x[:, lo], x[:, lo + h] = a + b, a - b
    assert not np.array_equal(fwd, x * np.float32(0.25))


def test_non_finite_rejected():
    with pytest.raises(ValueError):
        orc.quantize(np.array([1.0, np.inf], dtype=np.float32), 8)


STOCH = [c for c in MANIFEST["cases"] if c.startswith("stoch")]


@pytest.mark.parametrize("case", STOCH)
def test_stochastic_case_bit_exact(case):
    """True stochastic rounding (RngState / Philox draws, quantize.py:114-125)."""
    g = load(case)
    st = {}
    gx, gw = orc.hlq_backward(g["x"], g["w"], g["gy"], bases=tuple(g["bases"]),
                              bits_gx=int(g["bits_gx"]), bits_gw=int(g["bits_gw"]), stages=st,
                              rng=int(g["rng_seed"]))
    for key in ("gx_codes_g", "gx_codes_w", "x_codes", "gw_codes_g"):
        assert np.array_equal(st[key], g[key]), key
    for key in ("gx_scale_g", "gx_scale_w", "x_scale", "gw_scale_g"):
        assert np.float32(st[key]).tobytes() == np.float32(g[key]).tobytes(), key
    assert np.array_equal(gx, g["gx"]) and np.array_equal(gw, g["gw"])


def test_rng_split_matches_reference_values():
    """splitmix64 splits (quantize.py:48-52): values taken from the reference's
    RngState in the build container; the package mirror and the oracle agree."""
    from paper_2406_15102_b200.rng import RngState, site_key
    assert RngState(5).split(21).seed == 14007819075902455836
    for seed in (0, 7, 0x1234ABCD, 2 ** 64 - 1):
        for tag in (11, 12, 21, 22):
            assert site_key(RngState(seed), tag) == (orc.split_seed(seed, tag), 0)


CONTAINERS = [c for c in MANIFEST["cases"] if c.startswith("acbp_")]


@pytest.mark.parametrize("case", CONTAINERS)
def test_container_bytes_match_reference(case):
    """oracle.acbp_container == the reference's acbp_pack bytes."""
    g = load(case)
    x = g["x"]
    B, L, I = x.shape
    bits = int(g["bits"])
    bases = tuple(int(b) for b in g["bases"])
    if B == 0:
        payload, scale = g["payload"], g["scale"]
    else:
        payload, scale, axis = orc.acbp_compress(x, bases, bits, pad_small_axes=bool(g["pad_small"]))
        assert axis == int(g["axis"])
        assert np.array_equal(payload.reshape(-1), g["payload"].reshape(-1))
    buf = orc.acbp_container(payload, bits, 16, bases, B, L, I, scale)
    assert buf == g["container"].tobytes()


CALIB = [c for c in MANIFEST["cases"] if c.startswith("calib_")]


@pytest.mark.parametrize("case", CALIB)
def test_calibration_matches_reference(case):
    g = load(case)
    e = orc.basis_energy(g["gy"], int(g["axis"]))
    assert np.array_equal(np.abs(e).mean(axis=0), g["means"])
    assert orc.select_bases(e, int(g["rank"])) == tuple(int(b) for b in g["bases"])


BASELINES = [c for c in MANIFEST["cases"] if c.startswith("base_")]


def _baseline_args(g):
    bits = lambda v: None if int(v) == 0 else int(v)  # noqa: E731
    seed = int(g["rng_seed"])
    return dict(gx_mode=str(g["gx_mode"]), gx_bits=bits(g["gx_bits"]), gw_mode=str(g["gw_mode"]),
                gw_bits=bits(g["gw_bits"]), bases=tuple(int(b) for b in g["bases"]),
                pad_small_axes=bool(g["pad_small"]), rng=None if seed < 0 else seed)


def _is_int(mode, bits):
    return mode in ("quant", "ht_quant", "lowrank_quant") and bits is not None


@pytest.mark.parametrize("case", BASELINES)
def test_baseline_strategies_match_reference(case):
    """Oracle restatement of every baseline mode vs the reference's
    strategy_backward: integer paths bit-exact, float paths to fp32 roundoff."""
    g = load(case)
    a = _baseline_args(g)
    gx, gw = orc.strategy_backward(g["x"], g["w"], g["gy"], **a)
    for got, ref, mode, bits in ((gx, g["gx"], a["gx_mode"], a["gx_bits"]),
                                 (gw, g["gw"], a["gw_mode"], a["gw_bits"])):
        assert got.shape == ref.shape and got.dtype == ref.dtype
        if _is_int(mode, bits):
            assert np.array_equal(got, ref)
        else:
            assert np.allclose(got, ref, rtol=1e-5, atol=1e-6 * float(np.abs(ref).max() + 1e-30))
