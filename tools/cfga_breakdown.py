import sys, torch
sys.path.insert(0, '.')
import bench
from paper_2406_15102_b200.backprop import BackwardStrategy
from paper_2406_15102_b200.hadamard import HadamardPlan, lowest_sequency_bases
flush = torch.empty(64 * 1024 * 1024, device="cuda")
T, I, O = 4096, 1024, 1024
x = torch.randn(T, I, device="cuda"); gy = torch.randn(T, O, device="cuda") * 1e-3
for r in (2, 8):
    strat = BackwardStrategy.hlq().with_plan(HadamardPlan(basis_indices=lowest_sequency_bases(16, r)))
    h, d = bench._linear_pair(torch, I, O, strat)
    out = bench.layer_autograd(torch, flush, h, None, x, gy, amp=False)
    print(r, out['hlq_bwd_us'], out['hlq_fwd_us'], out['acbp_fwd_us'], out['libhlq_bwd_us'], out['libhlq_bwd_kernels'])
