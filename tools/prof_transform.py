"""ncu driver: the STATS and QUANT passes of the dual transform at one shape."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2406_15102_b200 import ops  # noqa: E402

B, L, I, O = (int(v) for v in (sys.argv[1] if len(sys.argv) > 1 else "128,197,768,3072").split(","))
gy = (torch.randn(B, L, O, device="cuda") * 1e-3).to(torch.bfloat16)
k = ops.proj_rows_k(B, L, 8)
cgx = torch.empty(B * L, ops.pad16(O), dtype=torch.int8, device="cuda")
cgw = torch.empty(O, max(ops.pad16(k), 16), dtype=torch.int8, device="cuda")
sc = torch.empty(2, device="cuda")
st = ops.new_stats("cuda")
for _ in range(2):
    st.zero_()
    ops.transform_pass(gy, B, L, O, O, L * O, True, True, 0x5555, 4, 8, 0, st)
    ops.transform_pass(gy, B, L, O, O, L * O, True, True, 0x5555, 4, 8, 1, st, cgx, cgw, sc[0:1], sc[1:2])
torch.cuda.synchronize()
