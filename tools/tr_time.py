"""Device time of the training path's transform calls at the ViT-B/16 shapes
(batch 128, bf16): the fused dual gy transform with the bias-gradient column
sums (every Linear's backward) and the forward ACBP of X, CUDA events, L2
flushed, median of 20 (development A/B tool).

    python tools/tr_time.py [--reps 20]
"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2406_15102_b200 import ops  # noqa: E402


def dev_us(fn, flush, reps):
    ts = []
    for i in range(reps + 2):
        flush.zero_()
        torch.cuda._sleep(1_000_000)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        e.synchronize()
        if i >= 2:
            ts.append(s.elapsed_time(e) * 1e3)
    return sorted(ts)[len(ts) // 2]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--dist", default="normal", choices=["normal", "lognormal"],
                    help="gy distribution: N(0,1)*1e-3 or SURVEY 8(d)'s lognormal(0,1.4)*sign*1e-3")
    a = ap.parse_args()
    flush = torch.empty(64 * 1024 * 1024, device="cuda")
    B, L = 128, 197
    out = {}
    for O in (768, 2304, 3072):
        if a.dist == "normal":
            gy = (torch.randn(B, L, O, device="cuda") * 1e-3).to(torch.bfloat16)
        else:
            z = torch.randn(B, L, O, device="cuda")
            gy = (torch.exp(1.4 * torch.randn_like(z)) * torch.sign(z) * 1e-3).to(torch.bfloat16)
        out[f"dual_cs_{O}"] = round(dev_us(lambda: ops.quant_dual(gy, B, L, O, 0x5555, 4, 8, O, L * O, colsum=True),
                                           flush, a.reps), 1)
    for I in (768, 3072):
        x = torch.randn(B, L, I, device="cuda").to(torch.bfloat16)
        out[f"acbp_{I}"] = round(dev_us(lambda: ops.quant_proj_rows(x, B, L, I, 0x5555, 8, I, L * I), flush, a.reps), 1)
    ws = [torch.randn(o, i, device="cuda") * (2.0 / i) ** 0.5
          for o, i in [(2304, 768), (768, 768), (3072, 768), (768, 3072)] * 12 + [(1000, 768)]]
    out["wcodes_49"] = round(dev_us(lambda: ops.quant_weights(ws, 4, bf16=True), flush, a.reps), 1)
    out["dist"] = a.dist
    print(json.dumps(out))


if __name__ == "__main__":
    main()
