"""CPU-side checks: the C-ABI library loads and exports every declared symbol,
host-side configuration mirrors the reference, and the product path refuses
to run without CUDA (there is no CPU fallback)."""
import json
import os
import re
import subprocess

import numpy as np
import pytest
import torch

import paper_2406_15102_b200 as h
from paper_2406_15102_b200 import _lib, ops

from .conftest import GOLDEN, ROOT

HEADER = os.path.join(ROOT, "include", "hlq_b200.h")


def declared_symbols():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"HLQ_API\s+[\w\s\*]+?\b(hlq_\w+)\s*\(", src)))


def test_library_built_and_loads():
    assert os.path.exists(_lib.LIB_PATH), "run python -m paper_2406_15102_b200.build"
    assert _lib.version().startswith("hlq_b200")


def test_every_header_symbol_exported():
    decl = declared_symbols()
    assert len(decl) >= 15
    lib = _lib.load()
    for name in decl:
        assert hasattr(lib, name), name
    assert sorted(_lib.exported_symbols()) == decl
    nm = subprocess.run(["nm", "-D", _lib.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (hlq_\w+)", nm))
    assert set(decl) <= exported


def test_library_is_sm100a_tcgen05():
    sass = subprocess.run(["cuobjdump", "-sass", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "UTCIMMA" in sass, "int8 GEMM must use tcgen05 (UTCIMMA)"
    assert "UTMALDG" in sass, "GEMM operands must be staged by TMA"
    assert "LDTM" in sass, "epilogue must read TMEM"
    assert "HMMA" not in sass and "IMMA.16" not in sass


def test_geometry_helpers_pure_c():
    lib = _lib.load()
    assert lib.hlq_acbp_k(128, 197, 1, 8) == 128 * 13 * 8
    assert lib.hlq_acbp_k(4096, 1, 0, 2) == 256 * 2
    assert lib.hlq_acbp_rows(7, 40, 0) == 280 and lib.hlq_acbp_rows(7, 40, 1) == 40
    assert lib.hlq_hq_grad_input_ws(4096, 1000, 1024) >= 4096 * 1008 + 1024 * 1008
    assert lib.hlq_device_ok() in (0, 1)


def test_status_codes_map_to_reference_exceptions():
    with pytest.raises(h.DimensionError):
        _lib.check(_lib.HLQ_ERR_DIMENSION)
    with pytest.raises(h.ParameterError):
        _lib.check(_lib.HLQ_ERR_PARAMETER)
    with pytest.raises(h.StateError):
        _lib.check(_lib.HLQ_ERR_STATE)
    with pytest.raises(ValueError):
        _lib.check(_lib.HLQ_ERR_NONFINITE)
    # C-side validation runs before any CUDA call
    lib = _lib.load()
    st = lib.hlq_gemm_i8(None, 16, None, 16, 16, 16, 140000, 8, 8, None, None, 1.0, 0, None, 0, 16,
                         None, 16, None)
    assert st in (_lib.HLQ_ERR_DIMENSION, _lib.HLQ_ERR_PARAMETER)
    st = lib.hlq_gemm_i8(None, 16, None, 16, 16, 16, 16, 3, 8, None, None, 1.0, 0, None, 0, 16, None,
                         16, None)
    assert st == _lib.HLQ_ERR_PARAMETER and b"bits" in lib.hlq_last_error()


def test_no_cpu_fallback():
    x = torch.zeros((2, 32, 16))
    with pytest.raises(h.ParameterError, match="CUDA"):
        h.acbp_compress(x, h.HadamardPlan())
    with pytest.raises(h.ParameterError):
        ops.quant_ht_cols(torch.zeros(4, 16), 4)


def test_plan_and_bases_match_reference():
    ref = json.load(open(os.path.join(GOLDEN, "bases16.json")))
    for r, idx in ref.items():
        assert list(h.lowest_sequency_bases(16, int(r))) == idx
    p = h.HadamardPlan()
    assert p.rank == 8 and p.basis_bitmap() == 0x5555
    assert h.HadamardPlan().with_rank(2).basis_bitmap() == 0x0101
    assert h.HadamardPlan.from_bitmap(16, 0x5555) == p
    with pytest.raises(h.ParameterError):
        h.HadamardPlan(block_size=12)
    with pytest.raises(h.ParameterError):
        h.HadamardPlan(basis_indices=(3, 1))
    with pytest.raises(h.ParameterError):
        h.HadamardPlan(block_size=8, basis_indices=(0, 2)).gpu_bitmap()


def test_strategy_mirror():
    s = h.BackwardStrategy.hlq()
    assert s.grad_input_path == h.PathSpec("ht_quant", 4)
    assert s.grad_weight_path == h.PathSpec("lowrank_quant", 8)
    assert s.uses_compressed_activation
    w8 = s.with_warmup_bits(8)
    assert w8.grad_input_path.bits == 8 and w8.plan == s.plan
    with pytest.raises(h.ParameterError):
        h.BackwardStrategy("x", h.PathSpec("fp", 4), h.PathSpec("fp"))
    with pytest.raises(h.ParameterError):
        h.BackwardStrategy("x", h.PathSpec("ht_quant", 3), h.PathSpec("fp"))


def test_axis_rule():
    assert h.ht_axis_for(4, 32, 16) == 1
    assert h.ht_axis_for(32, 4, 16) == 0
    with pytest.raises(h.DimensionError):
        h.ht_axis_for(4, 8, 16)
    assert h.ht_axis_for(4, 8, 16, pad_small_axes=True) == 1
    assert h.ht_axis_for(8, 4, 16, pad_small_axes=True) == 0


def test_reference_payload_reindexing_matches_oracle_layout():
    """The K-major batch-axis payload (rows l*I + i) maps back onto the
    reference's (blk*r + j)*L + l rows -- checked on the oracle's own codes."""
    from oracle import hlq_oracle as orc
    rng = np.random.default_rng(3)
    B, L, I = 32, 3, 5
    x = rng.standard_normal((B, L, I)).astype(np.float32)
    codes, scale, axis = orc.acbp_compress(x, orc.lowest_sequency_bases(16, 8))
    assert axis == 0
    q = codes.shape[0] // L
    kmajor = codes.reshape(q, L, I).transpose(1, 2, 0).reshape(L * I, q)   # what the kernel writes
    acbp = h.ACBPActivation(h.QuantizedTensor(torch.from_numpy(kmajor), 8, torch.tensor([scale])),
                            (B, L, I), 0, h.HadamardPlan(), q)
    assert np.array_equal(acbp.reference_payload().numpy(), codes)


def test_bench_reference_arm_contract():
    """`bench.py --impl reference` (the reference algorithm on the host cores)
    prints one JSON line with the bench contract's keys; it needs no GPU."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--impl", "reference", "--steps", "1",
                          "--warmup", "0"], capture_output=True, text=True, timeout=600, cwd=root)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    for k in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert k in line, k
    assert line["impl"] == "reference" and line["value"] > 0 and line["unit"] == "img/s"
    # the unmodified reference staged into oracle/_ref (oracle/stage_ref.sh), else the numpy port
    staged = os.path.isfile(os.path.join(root, "oracle", "_ref", "hlq", "backprop.py"))
    assert line["cpu_baseline"]["kind"] == ("reference" if staged else "port")
    assert line["cpu_baseline"]["value"] == line["value"]
    # ms_per_step is the measured wall time of one step (the driver's fit check)
    assert 0 < line["ms_per_step"] < 60_000
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["value"] == line["value"]
    with open(os.path.join(root, "BASELINE.json")) as f:
        assert line["metric"] == json.load(f)["metric"]
