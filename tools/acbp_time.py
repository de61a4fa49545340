"""Dev: ACBP container pack / unpack at the ViT-B/16 fc1 input (10.2 MB):
kernel breakdown (torch.profiler / CUPTI) and wall time per call."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2406_15102_b200 import HadamardPlan, acbp_compress  # noqa: E402
from paper_2406_15102_b200 import acbp as acbp_mod  # noqa: E402

xa = torch.randn(128, 197, 768, device="cuda", dtype=torch.bfloat16)
act = acbp_compress(xa, HadamardPlan())
buf = acbp_mod.acbp_pack(act)
for _ in range(3):
    acbp_mod.acbp_unpack(acbp_mod.acbp_pack(act))
torch.cuda.synchronize()
for name, fn in (("pack", lambda: acbp_mod.acbp_pack(act)), ("unpack", lambda: acbp_mod.acbp_unpack(buf))):
    t0 = time.perf_counter()
    for _ in range(20):
        fn()
    torch.cuda.synchronize()
    print(f"{name}: wall {1e6 * (time.perf_counter() - t0) / 20:.1f} us per call, {buf.numel()} bytes")
    with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
        for _ in range(5):
            fn()
        torch.cuda.synchronize()
    for ev in sorted(prof.key_averages(), key=lambda e: -e.device_time_total)[:8]:
        if ev.device_time_total > 0:
            print(f"   {ev.device_time_total / 5:8.1f} us/call  {ev.key[:90]}")
