"""Dev: torch.profiler kernel breakdown of the HLQ ResNet-18 CIFAR step."""
import collections
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2406_15102_b200.resnet import convert_resnet, resnet18_cifar  # noqa: E402

F = torch.nn.functional
torch.backends.cudnn.benchmark = True
x = torch.randn(256, 3, 32, 32, device="cuda").to(memory_format=torch.channels_last)
y = torch.randint(0, 10, (256,), device="cuda")
m = convert_resnet(resnet18_cifar().cuda().to(memory_format=torch.channels_last))
opt = torch.optim.SGD(m.parameters(), lr=1e-2, momentum=0.9, foreach=True)


def step():
    with torch.autocast("cuda", dtype=torch.bfloat16):
        loss = F.cross_entropy(m(x).float(), y)
    loss.backward()
    opt.step()
    opt.zero_grad(set_to_none=True)


for _ in range(5):
    step()
torch.cuda.synchronize()
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
    step()
    torch.cuda.synchronize()
agg = collections.defaultdict(lambda: [0, 0.0])
for ev in prof.events():
    if ev.device_type == torch.autograd.DeviceType.CUDA:
        n = ev.name
        for k in ("tma_tile_kernel<float", "tma_tile_kernel<__nv_bfloat16, 2, 0", "tma_tile_kernel<__nv_bfloat16, 2, 1",
                  "gemm_i8_2sm", "gemm_i8_kernel", "col2im", "im2col_proj", "tile_kernel", "splitk", "weight_codes"):
            if k in n:
                n = k
                break
        agg[n[:100]][0] += 1
        agg[n[:100]][1] += ev.device_time_total
tot = sum(v[1] for v in agg.values())
print(f"total {tot:.0f} us")
for k, (c, us) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:25]:
    print(f"{us:8.0f} us {c:4d}x {k}")
