"""Dev microbench: the ViT-B/16 transform launches of one training step at
their real shapes (CUDA-graph replays, L2 flushed), plus the torch bias-grad
reduction the fused column sums replace.  One JSON line.

    python tools/tr_shapes.py [--tag name]
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
    ap.add_argument("--tag", default="")
    a = ap.parse_args()
    B, L = 128, 197
    flush = torch.empty(64 * 1024 * 1024, device="cuda")
    res = {"tag": a.tag}
    for O in (3072, 2304, 768):
        gy = (torch.randn(B, L, O, device="cuda") * 1e-3).to(torch.bfloat16)
        res[f"dual_{O}"] = round(timeit(lambda: ops.quant_dual(gy, B, L, O, 0x5555, 4, 8, O, L * O),
                                        flush=flush), 1)
        res[f"dual_cs_{O}"] = round(timeit(lambda: ops.quant_dual(gy, B, L, O, 0x5555, 4, 8, O, L * O,
                                                                  colsum=True), flush=flush), 1)
        res[f"torch_sum_{O}"] = round(timeit(lambda: gy.reshape(-1, O).sum(0, dtype=torch.float32),
                                             flush=flush), 1)
    for I in (768, 3072):
        x = torch.randn(B, L, I, device="cuda").to(torch.bfloat16)
        res[f"proj_{I}"] = round(timeit(lambda: ops.quant_proj_rows(x, B, L, I, 0x5555, 8, I, L * I),
                                        flush=flush), 1)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
