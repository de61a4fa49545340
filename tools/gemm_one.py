"""Run one dX GEMM (int8 or packed A) a few times (for ncu)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2406_15102_b200 import ops  # noqa: E402

m, n, k = (int(v) for v in sys.argv[1].split(","))
packed = sys.argv[2] == "packed"
s = torch.tensor([0.01], device="cuda")
a = torch.randint(-7, 8, (m, ops.pad16(k)), dtype=torch.int8, device="cuda")
b = torch.randint(-7, 8, (n, ops.pad16(k)), dtype=torch.int8, device="cuda")
p = torch.randint(0, 256, (m, ops.packed_ld(k)), dtype=torch.uint8, device="cuda")
for _ in range(3):
    if packed:
        ops.gemm_i8(p, b, m, n, k, 4, 4, s, s, 1.0, exact=False, out_dtype=torch.bfloat16, a_packed=True)
    else:
        ops.gemm_i8(a, b, m, n, k, 4, 4, s, s, 1.0, exact=False, out_dtype=torch.bfloat16)
torch.cuda.synchronize()
