"""Dev: layer backward table + transform shapes in one JSON line (A/B builds via HLQ_LIB_PATH)."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402

t = bench.layer_bwd_table(torch)
print(json.dumps({"tag": sys.argv[1] if len(sys.argv) > 1 else "",
                  **{k: v["hlq_us"] for k, v in t.items() if isinstance(v, dict) and "hlq_us" in v},
                  **{k + "_fwd": v["fwd_overhead_us"] for k, v in t.items() if isinstance(v, dict) and "fwd_overhead_us" in v}}))
