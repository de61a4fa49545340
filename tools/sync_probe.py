"""Dev probe: ViT-B/16 HLQ step time with and without a per-step host sync,
plus allocator statistics (why does the un-synced loop run slower?)."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402


def main():
    torch.backends.cuda.matmul.allow_tf32 = True
    model = bench.make_model(torch, True)
    opt = torch.optim.SGD(model.parameters(), lr=1e-3, momentum=0.9, foreach=True)
    x = torch.randn(128, 3, 224, 224, device="cuda")
    y = torch.randint(0, 1000, (128,), device="cuda")
    bench.train_steps(torch, model, opt, x, y, 3)
    torch.cuda.synchronize()
    for mode in ("nosync", "sync", "nosync", "sync"):
        torch.cuda.reset_peak_memory_stats()
        st0 = torch.cuda.memory_stats()
        t0 = time.perf_counter()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(10):
            bench.train_steps(torch, model, opt, x, y, 1)
            if mode == "sync":
                torch.cuda.synchronize()
        e.record()
        torch.cuda.synchronize()
        st1 = torch.cuda.memory_stats()
        print(mode, f"{s.elapsed_time(e) / 10:.2f} ms/step", f"wall {(time.perf_counter() - t0) * 100:.2f} ms/step",
              "retries", st1["num_alloc_retries"] - st0["num_alloc_retries"],
              "cudaMalloc", st1.get("num_device_alloc", 0) - st0.get("num_device_alloc", 0),
              "cudaFree", st1.get("num_device_free", 0) - st0.get("num_device_free", 0),
              f"peak {torch.cuda.max_memory_allocated() / 2**30:.1f} GiB",
              f"reserved {torch.cuda.memory_reserved() / 2**30:.1f} GiB", flush=True)


if __name__ == "__main__":
    main()
