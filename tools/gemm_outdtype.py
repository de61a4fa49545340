import sys, os, json, torch
sys.path.insert(0, '/root/repo')
from paper_2406_15102_b200 import ops
from tools.tr_time import dev_us
flush = torch.empty(64 * 1024 * 1024, device="cuda")
s = torch.tensor([0.01], device="cuda")
out = {}
for (M, N, K) in [(25216, 3072, 768), (25216, 768, 3072), (25216*2, 3072, 768), (12608, 3072, 768), (25216, 3072, 384), (25216, 3072, 1536)]:
    a = torch.randint(-7, 8, (M, K), dtype=torch.int8, device="cuda")
    b = torch.randint(-7, 8, (N, K), dtype=torch.int8, device="cuda")
    r = {}
    r["bf16"] = round(dev_us(lambda: ops.gemm_i8(a, b, M, N, K, 4, 4, s, s, 1.0, exact=False, out_dtype=torch.bfloat16), flush, 10), 1)
    r["f32"] = round(dev_us(lambda: ops.gemm_i8(a, b, M, N, K, 4, 4, s, s, 1.0, exact=False, out_dtype=torch.float32), flush, 10), 1)
    r["tops_bf16"] = round(2 * M * N * K / r["bf16"] / 1e6)
    out[f"{M}x{N}x{K}"] = r
print(json.dumps(out))
