"""Dev tool: torch.profiler (CUPTI) kernel-time breakdown of the ViT-B/16
training step, HLQ vs dense bf16.

    python tools/step_profile.py [--batch 128]
"""
import argparse
import collections
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402


def profile(hlq: bool, batch: int):
    model = bench.make_model(torch, hlq)
    opt = torch.optim.SGD(model.parameters(), lr=1e-3, momentum=0.9, foreach=True)
    x = torch.randn(batch, 3, 224, 224, device="cuda")
    y = torch.randint(0, 1000, (batch,), device="cuda")
    bench.train_steps(torch, model, opt, x, y, 3)
    torch.cuda.synchronize()
    with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
        bench.train_steps(torch, model, opt, x, y, 2)
        torch.cuda.synchronize()
    agg = collections.defaultdict(lambda: [0, 0.0])
    for ev in prof.events():
        if ev.device_type == torch.autograd.DeviceType.CUDA:
            name = ev.name
            for key in ("tma_tile_kernel", "gemm_i8_kernel", "splitk_finalize", "tile_kernel", "im2col"):
                if key in name:
                    name = key
            a = agg[name[:90]]
            a[0] += 1
            a[1] += ev.device_time_total / 2 / 1e3
    tot = sum(v[1] for v in agg.values())
    print(f"=== {'HLQ' if hlq else 'dense'}: summed kernel time per step {tot:.2f} ms")
    for k, (n, ms) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:25]:
        print(f"{ms:8.3f} ms {n // 2:5d}x  {k}")
    del model, opt
    torch.cuda.empty_cache()


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=128)
    a = ap.parse_args()
    torch.backends.cuda.matmul.allow_tf32 = True
    profile(True, a.batch)
    profile(False, a.batch)
