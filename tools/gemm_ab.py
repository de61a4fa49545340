"""Device time of the dX GEMM with int8 vs packed int4 A (development A/B)."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2406_15102_b200 import ops  # noqa: E402
from tools.tr_time import dev_us  # noqa: E402


def main():
    flush = torch.empty(64 * 1024 * 1024, device="cuda")
    out = {}
    s = torch.tensor([0.01], device="cuda")
    for (m, n, k) in [(25216, 768, 3072), (25216, 3072, 768), (25216, 768, 2304), (25216, 768, 768)]:
        a = torch.randint(-7, 8, (m, ops.pad16(k)), dtype=torch.int8, device="cuda")
        b = torch.randint(-7, 8, (n, ops.pad16(k)), dtype=torch.int8, device="cuda")
        p = torch.randint(0, 256, (m, ops.packed_ld(k)), dtype=torch.uint8, device="cuda")
        i8 = dev_us(lambda: ops.gemm_i8(a, b, m, n, k, 4, 4, s, s, 1.0, exact=False, out_dtype=torch.bfloat16), flush, 10)
        i4 = dev_us(lambda: ops.gemm_i8(p, b, m, n, k, 4, 4, s, s, 1.0, exact=False, out_dtype=torch.bfloat16,
                                        a_packed=True), flush, 10)
        out[f"{m}x{n}x{k}"] = {"int8_us": round(i8, 1), "packed_us": round(i4, 1)}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
