"""Dev sweep: dW / dX GEMM time vs tile width and split count (HLQ_GEMM_BN /
HLQ_GEMM_SPLITS are read per call by the library's planner).

    python tools/gemm_sweep.py
"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2406_15102_b200 import ops  # noqa: E402
from tools.stage_bench import timeit  # noqa: E402


def main():
    flush = torch.empty(64 * 1024 * 1024, device="cuda")
    sa = torch.tensor([0.01], device="cuda")
    for name, M, N, K in [("proj_dw", 768, 768, 13312), ("fc1_dw", 3072, 768, 13312),
                          ("fc2_dw", 768, 3072, 13312), ("qkv_dw", 2304, 768, 13312),
                          ("fc1_dx", 25216, 768, 3072), ("fc2_dx", 25216, 3072, 768)]:
        a = torch.randint(-127, 128, (M, K), dtype=torch.int8, device="cuda")
        b = torch.randint(-127, 128, (N, K), dtype=torch.int8, device="cuda")
        res = {}
        for pair in ("0", "1"):
          for bn in ("128", "192", "256") if pair == "1" else ("128", "256"):
            for s in ("1", "2", "4"):
                if name.endswith("dx") and s != "1":
                    continue
                os.environ["HLQ_GEMM_BN"], os.environ["HLQ_GEMM_SPLITS"] = bn, s
                os.environ["HLQ_GEMM_PAIR"] = pair
                us = timeit(lambda: ops.gemm_i8(a, b, M, N, K, 8, 8, sa, sa, 1.0, exact=False,
                                                out_dtype=torch.bfloat16 if name.endswith("dx") else torch.float32),
                            iters=10, flush=flush)
                res[f"{'p' if pair == '1' else 'c'}{bn}_s{s}"] = round(us, 1)
        os.environ.pop("HLQ_GEMM_BN")
        os.environ.pop("HLQ_GEMM_SPLITS")
        os.environ.pop("HLQ_GEMM_PAIR")
        res["auto"] = round(timeit(lambda: ops.gemm_i8(a, b, M, N, K, 8, 8, sa, sa, 1.0, exact=False,
                                                       out_dtype=torch.bfloat16 if name.endswith("dx") else torch.float32),
                                   iters=10, flush=flush), 1)
        res["torch_int_mm"] = round(timeit(lambda: torch._int_mm(a, b.t()), iters=10, flush=flush), 1) \
            if M % 8 == 0 and N % 8 == 0 and K % 8 == 0 else None
        best = min(res, key=res.get)
        print(json.dumps({"gemm": name, "MNK": [M, N, K], "tops_best": round(2 * M * N * K / res[best] / 1e6, 1),
                          "best": best, **res}), flush=True)


if __name__ == "__main__":
    main()
