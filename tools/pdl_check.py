"""Dev: fused-transform scales against the oracle with many launches queued
(no host syncs in between): caller scratch (memset + launch) vs library slots."""
import sys

import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from oracle import hlq_oracle as orc  # noqa: E402
from paper_2406_15102_b200 import ops  # noqa: E402

torch.manual_seed(0)
B, L, O = 8, 197, 768
gys = [(torch.randn(B, L, O, device="cuda") * (10.0 ** -(i % 5))).to(torch.bfloat16) for i in range(6)]
want = []
for g in gys:
    gf = g.float().cpu().numpy()
    want.append(float(orc.quantize(orc.transform_axis(gf.reshape(B * L, O), 1, 16), 4)[1]))
for mode in ("caller", "pooled", "mixed"):
    outs = []
    for rep in range(10):
        for i, g in enumerate(gys):
            ws = mode == "caller" or (mode == "mixed" and (rep + i) % 2 == 0)
            outs.append((i, ops.quant_dual(g, B, L, O, 0x5555, 4, 8, O, L * O, colsum=True, want_stats=ws)[1]))
    torch.cuda.synchronize()
    bad = sum(float(s) != want[i] for i, s in outs)
    print(f"{mode}: {bad} of {len(outs)} scales differ from the oracle")
