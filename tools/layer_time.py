"""Dev: bench.py's per-layer table alone (ViT-B/16 shapes through the autograd
modules): HLQ vs dense backward per layer, and the libhlq kernels inside."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402

t = bench.layer_bwd_table(torch)
out = {n: {"hlq_bwd": t[n]["hlq_bwd_us"], "dense_bwd": t[n]["dense_bwd_us"], "speedup": t[n]["bwd_speedup"],
           "kernels": {k: v["us"] for k, v in t[n]["libhlq_bwd_kernels"].items()}}
       for n in ("qkv", "proj", "fc1", "fc2")}
out["block_bwd_speedup"] = t["block_total"]["bwd_speedup"]
out["knobs"] = {k: v for k, v in os.environ.items() if k.startswith("HLQ_")}
print(json.dumps(out))
