"""Dev: the GPU timeline around one fused transform launch (torch.profiler):
memset (caller scratch, `stats` argument) or library slot, kernel, gaps."""
import sys, torch
sys.path.insert(0, '/root/repo')
from paper_2406_15102_b200 import ops
B, L, O = 128, 197, 768
gy = (torch.randn(B, L, O, device="cuda") * 1e-3).to(torch.bfloat16)
for _ in range(3): ops.quant_dual(gy, B, L, O, 0x5555, 4, 8, O, L * O, colsum=True)
torch.cuda.synchronize()
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
    for _ in range(5):
        torch.cuda._sleep(200000)
        ops.quant_dual(gy, B, L, O, 0x5555, 4, 8, O, L * O, colsum=True, want_stats=False)
    torch.cuda.synchronize()
evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
evs.sort(key=lambda e: e.time_range.start)
prev = None
for e in evs[-12:]:
    st, en = e.time_range.start, e.time_range.end
    gap = (st - prev) if prev else 0
    print(f"{e.name[:60]:60s} dur {en-st:7.1f} us  gap {gap:7.1f}")
    prev = en
