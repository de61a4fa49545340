"""Per-stage CUDA-event timing of the HLQ backward at one layer shape vs the
dense bf16 backward (cuBLAS) of the same layer.  Dev tool; bench.py is the
contract benchmark.

    python tools/stage_bench.py --shape 128,197,768,3072 --dtype bf16
"""
from __future__ import annotations

import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2406_15102_b200 import ops  # noqa: E402
from paper_2406_15102_b200.backprop import _proj_view  # noqa: E402


def timeit(fn, iters=20, warmup=3, flush=None):
    """Median GPU time (us) of fn, captured in a CUDA graph so host overhead
    (ctypes, allocator) is excluded; L2 flushed before every replay."""
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        fn()
    for _ in range(2):
        g.replay()
    torch.cuda.synchronize()
    ts = []
    for _ in range(iters):
        if flush is not None:
            flush.zero_()
            flush[: 40 * 1024 * 1024].sum()  # evict the dirty lines before timing
        s = torch.cuda.Event(enable_timing=True)
        e = torch.cuda.Event(enable_timing=True)
        s.record()
        g.replay()
        e.record()
        e.synchronize()
        ts.append(s.elapsed_time(e) * 1e3)
    ts.sort()
    return ts[len(ts) // 2]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shape", default="128,197,768,3072", help="B,L,I,O")
    ap.add_argument("--dtype", default="bf16")
    ap.add_argument("--rank", type=int, default=8)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    B, L, I, O = (int(v) for v in a.shape.split(","))
    dt = torch.bfloat16 if a.dtype == "bf16" else torch.float32
    dev = "cuda"
    torch.manual_seed(0)
    x = torch.randn(B, L, I, device=dev).to(dt)
    w = (torch.randn(O, I, device=dev) * (2.0 / I) ** 0.5)
    gy = (torch.randn(B, L, O, device=dev) * 1e-3).to(dt)
    flush = torch.empty(256 * 1024 * 1024 // 4, device=dev)  # 256 MiB > L2
    T = B * L
    axis = 1 if L >= 16 else 0
    bitmap = {8: 0x5555, 2: 0x0101, 4: 0x1111, 16: 0xFFFF}[a.rank]
    res = {}
    segs, rows, cols, ld, sg = _proj_view(B, L, I, axis)
    res["acbp_x"] = timeit(lambda: ops.quant_proj_rows(x, segs, rows, cols, bitmap, 8, ld, sg), flush=flush)
    xp, k, sx, _ = ops.quant_proj_rows(x, segs, rows, cols, bitmap, 8, ld, sg)
    segs, rows, cols, ld, sgo = _proj_view(B, L, O, axis)
    res["proj_gy"] = timeit(lambda: ops.quant_proj_rows(gy, segs, rows, cols, bitmap, 8, ld, sgo), flush=flush)
    cg, kg, sgw, _ = ops.quant_proj_rows(gy, segs, rows, cols, bitmap, 8, ld, sgo)
    res["ht_gy"] = timeit(lambda: ops.quant_ht_cols(gy.reshape(T, O), 4), flush=flush)
    cgx, sgx, _ = ops.quant_ht_cols(gy.reshape(T, O), 4)
    res["ht_w"] = timeit(lambda: ops.quant_proj_rows(w, 1, O, I, 0xFFFF, 4), flush=flush)
    cw, _, sw, _ = ops.quant_proj_rows(w, 1, O, I, 0xFFFF, 4)
    groups = L if axis == 0 else 1
    res["gemm_dw"] = timeit(lambda: ops.gemm_i8(cg, xp, O, I, k, 8, 8, sgw, sx, 1.0, exact=False,
                                                groups=groups, a_gstride=cg.stride(0) * O,
                                                b_gstride=xp.stride(0) * I), flush=flush)
    res["gemm_dx"] = timeit(lambda: ops.gemm_i8(cgx, cw, T, I, ops.pad16(O), 4, 4, sgx, sw, 1.0,
                                                exact=False, out_dtype=dt), flush=flush)
    res["gemm_dx_exact_f32"] = timeit(lambda: ops.gemm_i8(cgx, cw, T, I, ops.pad16(O), 4, 4, sgx, sw,
                                                          1.0, exact=True), flush=flush)
    if axis == 1 or L == 1:
        res["dual_gy"] = timeit(lambda: ops.quant_dual(gy, segs, rows, cols, bitmap, 4, 8, ld, sgo),
                                flush=flush)
        res["dual_gy_GBps"] = (T * O * (2 if dt == torch.bfloat16 else 4) + T * ops.pad16(O) + O * kg) \
            / res["dual_gy"] / 1e3
        res["hlq_bwd_total"] = res["dual_gy"] + res["ht_w"] + res["gemm_dw"] + res["gemm_dx"]
    else:
        res["hlq_bwd_total"] = res["proj_gy"] + res["ht_gy"] + res["ht_w"] + res["gemm_dw"] + res["gemm_dx"]
    # dense bf16 backward of the same layer (cuBLAS): dX = gy W, dW = gy^T x
    xb, wb, gb = x.to(torch.bfloat16).reshape(T, I), w.to(torch.bfloat16), gy.to(torch.bfloat16).reshape(T, O)
    res["dense_dx"] = timeit(lambda: gb @ wb, flush=flush)
    res["dense_dw"] = timeit(lambda: gb.t() @ xb, flush=flush)
    res["dense_bwd_total"] = res["dense_dx"] + res["dense_dw"]
    # int8 cuBLASLt reference for the dX GEMM shape
    try:
        res["torch_int_mm_dx"] = timeit(lambda: torch._int_mm(cgx[:, :ops.pad16(O)], cw.t()), flush=flush)
    except Exception as e:  # noqa: BLE001
        res["torch_int_mm_dx"] = str(e)[:80]
    ops_gx = 2 * T * ops.pad16(O) * I
    ops_gw = 2 * k * I * O * groups
    res["gemm_dx_TOPS"] = ops_gx / res["gemm_dx"] / 1e6
    res["gemm_dw_TOPS"] = ops_gw / res["gemm_dw"] / 1e6
    el = 2 if dt == torch.bfloat16 else 4
    res["ht_gy_GBps"] = (T * O * el + T * ops.pad16(O)) / res["ht_gy"] / 1e3
    res["proj_gy_GBps"] = (T * O * el + O * kg) / res["proj_gy"] / 1e3
    res["acbp_x_GBps"] = (T * I * el + I * k) / res["acbp_x"] / 1e3
    res["speedup_vs_dense"] = res["dense_bwd_total"] / res["hlq_bwd_total"]
    res["shape"] = [B, L, I, O]
    res["dtype"] = a.dtype
    line = json.dumps({k: (round(v, 3) if isinstance(v, float) else v) for k, v in res.items()})
    print(line)
    if a.out:
        with open(a.out, "a") as f:
            f.write(line + "\n")


if __name__ == "__main__":
    main()
