"""Dev microbench of the transform kernels at one layer shape: the fused
single-launch dual quantizer vs its STATS and QUANT passes launched alone.

    python tools/transform_bench.py --shape 128,197,768,3072
"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2406_15102_b200 import ops  # noqa: E402
from tools.stage_bench import timeit  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shape", default="128,197,768,3072")
    ap.add_argument("--dist", default="normal", choices=["normal", "lognormal"])
    a = ap.parse_args()
    B, L, I, O = (int(v) for v in a.shape.split(","))
    flush = torch.empty(64 * 1024 * 1024, device="cuda")
    if a.dist == "normal":
        gy = (torch.randn(B, L, O, device="cuda") * 1e-3).to(torch.bfloat16)
    else:
        z = torch.randn(B, L, O, device="cuda")
        gy = (torch.exp(1.4 * torch.randn_like(z)) * torch.sign(z) * 1e-3).to(torch.bfloat16)
    k = ops.proj_rows_k(B, L, 8)
    cgx = torch.empty(B * L, ops.pad16(O), dtype=torch.int8, device="cuda")
    cgw = torch.empty(O, max(ops.pad16(k), 16), dtype=torch.int8, device="cuda")
    sc = torch.empty(2, device="cuda")
    st = ops.new_stats("cuda")
    res = {"shape": [B, L, I, O], "dist": a.dist}
    res["dual_fused"] = timeit(lambda: ops.quant_dual(gy, B, L, O, 0x5555, 4, 8, O, L * O), flush=flush)
    res["dual_fused_noflush"] = timeit(lambda: ops.quant_dual(gy, B, L, O, 0x5555, 4, 8, O, L * O))

    def stats():
        st.zero_()
        ops.transform_pass(gy, B, L, O, O, L * O, True, True, 0x5555, 4, 8, 0, st)

    def quant():
        ops.transform_pass(gy, B, L, O, O, L * O, True, True, 0x5555, 4, 8, 1, st, cgx, cgw, sc[0:1], sc[1:2])

    stats()
    res["stats_pass"] = timeit(stats, flush=flush)
    res["quant_pass"] = timeit(quant, flush=flush)
    res["quant_pass_noflush"] = timeit(quant)
    res["ht_only"] = timeit(lambda: ops.quant_ht_cols(gy.view(B * L, O), 4), flush=flush)
    res["proj_only"] = timeit(lambda: ops.quant_proj_rows(gy, B, L, O, 0x5555, 8, O, L * O), flush=flush)
    mb = gy.numel() * 2 / 1e6
    res["gy_MB"] = round(mb, 1)
    res["stats_GBps"] = round(mb / res["stats_pass"] * 1e3, 1)
    print(json.dumps({kk: (round(v, 1) if isinstance(v, float) else v) for kk, v in res.items()}))


if __name__ == "__main__":
    main()
