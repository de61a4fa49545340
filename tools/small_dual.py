"""Device time of the dual transform at the ResNet-18 CIFAR gy shapes (dev A/B)."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2406_15102_b200 import ops  # noqa: E402
from tools.tr_time import dev_us  # noqa: E402

flush = torch.empty(64 * 1024 * 1024, device="cuda")
out = {}
for (B, L, O) in [(256, 16, 512), (256, 64, 256), (256, 256, 128), (256, 1024, 64), (16, 256, 1024)]:
    g = (torch.randn(B, L, O, device="cuda") * 1e-3).to(torch.bfloat16)
    out[f"{B}x{L}x{O}"] = round(dev_us(lambda: ops.quant_dual(g, B, L, O, 0x5555, 4, 8, O, L * O, colsum=True),
                                       flush, 20), 1)
print(json.dumps(out))
