"""Tiny driver for ncu: runs one HLQ stage a few times at a layer shape.

    ncu --set full -k regex:tile_kernel -c 2 python tools/prof_driver.py dual 128,197,768,3072
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2406_15102_b200 import ops  # noqa: E402


def main():
    what = sys.argv[1]
    B, L, I, O = (int(v) for v in sys.argv[2].split(","))
    reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
    dt = torch.bfloat16
    torch.manual_seed(0)
    T = B * L
    x = torch.randn(B, L, I, device="cuda").to(dt)
    w = torch.randn(O, I, device="cuda") * (2.0 / I) ** 0.5
    gy = (torch.randn(B, L, O, device="cuda") * 1e-3).to(dt)
    axis = 1 if L >= 16 else 0
    segs, rows = (B, L) if axis == 1 else (1, B)
    xp, k, sx, _ = ops.quant_proj_rows(x, segs, rows, I, 0x5555, 8, I, L * I)
    cgx, sgx, cg, kg, sg, _ = ops.quant_dual(gy, segs, rows, O, 0x5555, 4, 8, O, L * O)
    cw, _, sw, _ = ops.quant_proj_rows(w, 1, O, I, 0xFFFF, 4)
    st = ops.new_stats("cuda")
    sc = torch.empty(2, device="cuda")
    for _ in range(reps):
        if what == "statspass":  # the fused kernel's two passes launched alone (dev A/B)
            st.zero_()
            ops.transform_pass(gy, segs, rows, O, O, L * O, True, True, 0x5555, 4, 8, 0, st)
        elif what == "quantpass":
            ops.transform_pass(gy, segs, rows, O, O, L * O, True, True, 0x5555, 4, 8, 1, st, cgx, cg,
                               sc[0:1], sc[1:2])
        elif what == "dual":
            ops.quant_dual(gy, segs, rows, O, 0x5555, 4, 8, O, L * O)
        elif what == "dualcs":  # as the training path runs it: with the bias-gradient column sums
            ops.quant_dual(gy, segs, rows, O, 0x5555, 4, 8, O, L * O, colsum=True)
        elif what == "acbp":
            ops.quant_proj_rows(x, segs, rows, I, 0x5555, 8, I, L * I)
        elif what == "w":
            ops.quant_proj_rows(w, 1, O, I, 0xFFFF, 4)
        elif what == "gemm_dx":
            ops.gemm_i8(cgx, cw, T, I, ops.pad16(O), 4, 4, sgx, sw, 1.0, exact=False, out_dtype=dt)
        elif what == "gemm_dw":
            ops.gemm_i8(cg, xp, O, I, k, 8, 8, sg, sx, 1.0, exact=False)
        elif what == "gemm_pair":  # dW + dX as the training path issues them (one CTA-pair launch)
            ops.gemm_i8_pair(dict(a=cg, b=xp, m=O, n=I, k=k, bits_a=8, bits_b=8, sa=sg, sb=sx),
                             dict(a=cgx, b=cw, m=T, n=I, k=ops.pad16(O), bits_a=4, bits_b=4, sa=sgx, sb=sw,
                                  out_dtype=dt))
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()
