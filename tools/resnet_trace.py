"""Dev: libhlq calls of one HLQ ResNet-18 CIFAR step by (operation, shape), CUDA events."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2406_15102_b200 import ops  # noqa: E402
from paper_2406_15102_b200.resnet import convert_resnet, resnet18_cifar  # noqa: E402

F = torch.nn.functional
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
with ops.trace() as tr:
    step()
s = tr.summary(by="key")
tot = sum(v["us"] for v in s.values())
print(f"libhlq total {tot:.0f} us")
for k, v in sorted(s.items(), key=lambda kv: -kv[1]["us"])[:30]:
    print(f"{v['us']:8.1f} us {v['calls']:3d}x  {k}")
