"""ncu driver: one int8 GEMM shape (env HLQ_GEMM_* select the variant)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2406_15102_b200 import ops  # noqa: E402

M, N, K = (int(v) for v in sys.argv[1].split(","))
a = torch.randint(-127, 128, (M, K), dtype=torch.int8, device="cuda")
b = torch.randint(-127, 128, (N, K), dtype=torch.int8, device="cuda")
s = torch.tensor([0.01], device="cuda")
for _ in range(3):
    ops.gemm_i8(a, b, M, N, K, 8, 8, s, s, 1.0, exact=False, out_dtype=torch.bfloat16)
torch.cuda.synchronize()
