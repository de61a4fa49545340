"""Dev: kernel breakdown of the HLQ conv backward at BASELINE config (b)."""
import collections
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2406_15102_b200.backprop import BackwardStrategy  # noqa: E402
from paper_2406_15102_b200.conv import _conv_backward, conv_acbp_compress  # noqa: E402

B, C, H, W, k = 128, 256, 14, 14, 3
xc = torch.randn(B, C, H, W, device="cuda").to(memory_format=torch.channels_last).to(torch.bfloat16)
w4 = torch.randn(C, C, k, k, device="cuda") * (2.0 / (C * k * k)) ** 0.5
gyc = (torch.randn(B, C, H, W, device="cuda") * 1e-3).to(torch.bfloat16).to(memory_format=torch.channels_last)
strat = BackwardStrategy.hlq()
for _ in range(3):
    acbp, _ = conv_acbp_compress(xc, k, 1, 1, strat)
    _conv_backward(acbp, w4, gyc, xc.shape, 1, 1, strat, 1.0, False, torch.bfloat16)
torch.cuda.synchronize()
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
    acbp, _ = conv_acbp_compress(xc, k, 1, 1, strat)
    _conv_backward(acbp, w4, gyc, xc.shape, 1, 1, strat, 1.0, False, torch.bfloat16)
    torch.cuda.synchronize()
for ev in prof.events():
    if ev.device_type == torch.autograd.DeviceType.CUDA:
        print(f"{ev.device_time_total:9.1f} us  {ev.name[:110]}")
