"""Dev: device time of the ViT-B/16 dX / dW GEMMs under the current planner
knobs (HLQ_GEMM_BN / HLQ_GEMM_SPLITS / HLQ_GEMM_PAIR are read once per
process, so sweep them across processes):

    for p in 0 1; do HLQ_GEMM_PAIR=$p python tools/gemm_time.py; done
"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2406_15102_b200 import ops  # noqa: E402
from tools.tr_time import dev_us  # noqa: E402

SHAPES = [("proj_dw", 768, 768, 13312), ("fc1_dw", 3072, 768, 13312), ("fc2_dw", 768, 3072, 13312),
          ("qkv_dw", 2304, 768, 13312), ("fc1_dx", 25216, 768, 3072), ("fc2_dx", 25216, 3072, 768),
          ("qkv_dx", 25216, 768, 2304), ("proj_dx", 25216, 768, 768)]


def main():
    flush = torch.empty(64 * 1024 * 1024, device="cuda")
    sa = torch.tensor([0.01], device="cuda")
    knobs = {k: v for k, v in os.environ.items() if k.startswith("HLQ_GEMM")}
    out = {"knobs": knobs}
    for name, M, N, K in SHAPES:
        a = torch.randint(-127, 128, (M, K), dtype=torch.int8, device="cuda")
        b = torch.randint(-127, 128, (N, K), dtype=torch.int8, device="cuda")
        dt = torch.bfloat16 if name.endswith("dx") else torch.float32
        out[name] = round(dev_us(lambda: ops.gemm_i8(a, b, M, N, K, 8, 8, sa, sa, 1.0, exact=False, out_dtype=dt),
                                 flush, 10), 1)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
