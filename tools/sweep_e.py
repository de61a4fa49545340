"""BASELINE config (e): HLQ Linear backward shape sweep on one B200.

    python tools/sweep_e.py [--out profiles/r02_sweep.jsonl] [--quick]

tokens T in {2K..64K} x hidden H in {768..8192} (square layers, I = O = H) x
rank r in {1, 2, 4, 8} x I/O dtype in {bf16, fp32}.  Each point runs the
product's autograd path (HLQLinear under convert_linears, 2-D input: the
projection runs along the token axis in 16-row blocks, like configs[0]) and
the dense bf16 nn.Linear backward on the same GPU; device time by CUDA events
with the host enqueue hidden behind a GPU spin, L2 flushed (bench.event_us).

Per point: HLQ backward us, the forward ACBP of X (the HLQ-only forward work)
us, dense bf16 forward / backward us, speedups (total = dense fwd + bwd vs
dense fwd + ACBP + HLQ bwd), and both roofline fractions of the HLQ backward
against SURVEY.md 8(d)'s algorithmic work (costmodel.py:194-198):
  ops   = 2*T*O_p*I (dX) + 2*K*I*O (dW), K = T*r/16
  bytes = T*O*s_in (gy) + O*I*4 (W) + K*I (payload) + T*I*s_out (dX) + O*I*4 (dW)
roofline time = max(bytes / HBM peak, ops / int8 peak); frac = that / measured.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r02_sweep.jsonl"))
    ap.add_argument("--quick", action="store_true", help="a handful of points (smoke)")
    a = ap.parse_args()
    import torch
    import bench
    from paper_2406_15102_b200.backprop import BackwardStrategy
    from paper_2406_15102_b200.hadamard import HadamardPlan, lowest_sequency_bases
    torch.backends.cuda.matmul.allow_tf32 = True
    peaks = bench.measured_peaks()
    int8 = bench.int8_peak_tops(torch)
    flush = torch.empty(64 * 1024 * 1024, device="cuda")
    tokens = [2048, 4096, 8192, 16384, 32768, 65536]
    hidden = [768, 1024, 2048, 4096, 8192]
    ranks = [1, 2, 4, 8]
    if a.quick:
        tokens, hidden, ranks = [4096], [1024], [2, 8]
    rows = []
    t0 = time.time()
    for T in tokens:
        for H in hidden:
            I = O = H
            torch.manual_seed(T + H)
            x32 = torch.randn(T, I, device="cuda")
            g32 = torch.randn(T, O, device="cuda") * 1e-3
            xb, gb = x32.to(torch.bfloat16), g32.to(torch.bfloat16)
            dense = None
            for r in ranks:
                strat = BackwardStrategy.hlq().with_plan(HadamardPlan(basis_indices=lowest_sequency_bases(16, r)))
                hnet, dense_m = bench._linear_pair(torch, I, O, strat)
                if dense is None:
                    d = bench.layer_autograd(torch, flush, hnet, dense_m, xb, gb, amp=True)
                    dense = (d["dense_bwd_us"], d["dense_fwd_us"])
                for io, (x, g, amp) in (("bf16", (xb, gb, True)), ("fp32", (x32, g32, False))):
                    h = bench.layer_autograd(torch, flush, hnet, None, x, g, amp=amp)
                    s = 2 if io == "bf16" else 4
                    K = T * r // 16
                    Op = (O + 15) // 16 * 16
                    ops_ = 2 * T * Op * I + 2 * K * I * O
                    nbytes = T * O * s + O * I * 4 + K * I + T * I * s + O * I * 4
                    t_hbm = nbytes / (peaks["hbm_gbs"] * 1e9) * 1e6
                    t_int8 = ops_ / (int8 * 1e12) * 1e6
                    roof = max(t_hbm, t_int8)
                    row = {"tokens": T, "hidden": H, "rank": r, "io": io, "K": K,
                           "hlq_bwd_us": h["hlq_bwd_us"], "acbp_fwd_us": h["acbp_fwd_us"],
                           "dense_bf16_bwd_us": dense[0], "dense_bf16_fwd_us": dense[1],
                           "bwd_speedup": round(dense[0] / h["hlq_bwd_us"], 3),
                           # the forward GEMM is the stock op in both arms: HLQ adds the ACBP of X
                           "total_speedup": round((dense[0] + dense[1]) / (dense[1] + h["acbp_fwd_us"] +
                                                                          h["hlq_bwd_us"]), 3),
                           "alg_bytes": nbytes, "alg_int8_ops": ops_,
                           "hbm_frac": round(t_hbm / h["hlq_bwd_us"], 4), "tensor_frac": round(t_int8 / h["hlq_bwd_us"], 4),
                           "roofline_frac": round(roof / h["hlq_bwd_us"], 4),
                           "bound": "hbm" if t_hbm >= t_int8 else "tensor",
                           "libhlq_bwd_us": h["libhlq_bwd_us"]}
                    rows.append(row)
                    print(json.dumps(row), flush=True)
                del hnet, dense_m
            del x32, g32, xb, gb
            torch.cuda.empty_cache()
    meta = {"meta": True, "hbm_gbs": peaks["hbm_gbs"], "hbm_source": peaks["source"], "int8_tops": round(int8, 1),
            "int8_source": "cuBLASLt torch._int_mm 8192^3 measured in this run", "points": len(rows),
            "wall_s": round(time.time() - t0, 1), "gpu": torch.cuda.get_device_name(0)}
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    with open(a.out, "w") as f:
        f.write(json.dumps(meta) + "\n")
        for r in rows:
            f.write(json.dumps(r) + "\n")
    print(json.dumps(meta))


if __name__ == "__main__":
    main()
