import os, sys, torch
sys.path.insert(0, "/root/repo")
from paper_2406_15102_b200 import ops
M, N, K = 512, 512, 1024
a = torch.randint(-127, 128, (M, K), dtype=torch.int8, device="cuda")
b = torch.randint(-127, 128, (N, K), dtype=torch.int8, device="cuda")
s1 = torch.tensor([1.0], device="cuda")
out, acc = ops.gemm_i8(a, b, M, N, K, 8, 8, s1, s1, 1.0, exact=True, want_acc=True)
torch.cuda.synchronize()
ref = (a.cpu().long() @ b.cpu().long().T)
print("pair probe equal:", torch.equal(acc.cpu().long(), ref), flush=True)
