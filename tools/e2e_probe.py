"""Dev: cost of the e2e pieces (per-step loss sync, H2D copies, prefetch)."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402

F = torch.nn.functional
model = bench.make_model(torch, True)
opt = torch.optim.SGD(model.parameters(), lr=1e-3, momentum=0.9, foreach=True)
x = torch.randn(128, 3, 224, 224, device="cuda")
y = torch.randint(0, 1000, (128,), device="cuda")
hx, hy = x.cpu().pin_memory(), y.cpu().pin_memory()


def run(kind, n=10):
    torch.cuda.synchronize()
    t = time.perf_counter()
    if kind == "prefetch":
        bench.train_steps(torch, model, opt, x, y, n, host=(hx, hy))
    else:
        for _ in range(n):
            if kind == "copy":
                x.copy_(hx, non_blocking=True)
                y.copy_(hy, non_blocking=True)
            with torch.autocast("cuda", dtype=torch.bfloat16):
                loss = F.cross_entropy(model(x).float(), y)
            loss.backward()
            opt.step()
            opt.zero_grad(set_to_none=True)
            if kind != "nosync":
                loss.item()
    torch.cuda.synchronize()
    return (time.perf_counter() - t) / n * 1e3


for kind in ("nosync", "sync", "copy", "prefetch"):
    run(kind, 5)
for r in range(2):
    print({k: round(run(k), 2) for k in ("nosync", "sync", "copy", "prefetch")})
