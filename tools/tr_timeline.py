"""Dev tool: per-CTA globaltimer timeline of the fused transform kernel (build
with -DHLQ_TR_TRACE into libhlq_b200_trace.so, load it via HLQ_LIB_PATH).

    HLQ_LIB_PATH=$PWD/paper_2406_15102_b200/libhlq_b200_trace.so python tools/tr_timeline.py
"""
import ctypes
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2406_15102_b200 import _lib, ops  # noqa: E402


def run(name, fn, buf):
    flush = torch.empty(64 * 1024 * 1024, device="cuda")
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    buf.fill_(0)
    flush.zero_()
    torch.cuda.synchronize()
    fn()
    torch.cuda.synchronize()
    t = buf.view(-1, 8).cpu()
    t = t[t[:, 0] > 0].double()
    t0 = t[:, 0].min()
    t = (t - t0) / 1e3  # us
    q = lambda v: f"{v.min():6.1f} {v.median():6.1f} {v.max():6.1f}"  # noqa: E731
    print(f"== {name}: {t.shape[0]} CTAs, span {t[:, 4].max():.1f} us")
    print(f"   start          {q(t[:, 0])}")
    print(f"   pass1 end      {q(t[:, 1])}   (pass1 dur {q(t[:, 1] - t[:, 0])})")
    print(f"   barrier exit   {q(t[:, 2])}")
    print(f"   pass2 end      {q(t[:, 3])}   (pass2 dur {q(t[:, 3] - t[:, 2])})")
    print(f"   end            {q(t[:, 4])}")


def main():
    lib = _lib.load()
    buf = torch.zeros(148 * 8 * 8, dtype=torch.int64, device="cuda")
    lib.hlq_debug_set_trace.argtypes = [ctypes.c_void_p]
    lib.hlq_debug_set_trace(ctypes.c_void_p(buf.data_ptr()))
    if len(sys.argv) > 1 and sys.argv[1] == "small":
        for B, L, O in [(256, 16, 512), (256, 64, 256), (256, 256, 128), (256, 1024, 64)]:
            gy = (torch.randn(B, L, O, device="cuda") * 1e-3).to(torch.bfloat16)
            run(f"dual {B}x{L}x{O}", lambda: ops.quant_dual(gy, B, L, O, 0x5555, 4, 8, O, L * O, colsum=True), buf)
        return
    if len(sys.argv) > 1 and sys.argv[1] == "config_a":
        T = 4096
        for bm in (0x0101, 0x5555):
            gy = torch.randn(T, 1024, device="cuda") * 1e-3
            run(f"config (a) dual fp32 bitmap {bm:#x}", lambda: ops.quant_dual(gy, 1, T, 1024, bm, 4, 8), buf)
            x = torch.randn(T, 1024, device="cuda")
            run(f"config (a) proj fp32 bitmap {bm:#x}", lambda: ops.quant_proj_rows(x, 1, T, 1024, bm, 8), buf)
        return
    B, L = 128, 197
    for I in (768, 3072):
        x = torch.randn(B, L, I, device="cuda").to(torch.bfloat16)
        run(f"proj {I}", lambda: ops.quant_proj_rows(x, B, L, I, 0x5555, 8, I, L * I), buf)
    for O in (768, 3072):
        gy = (torch.randn(B, L, O, device="cuda") * 1e-3).to(torch.bfloat16)
        run(f"dual {O}", lambda: ops.quant_dual(gy, B, L, O, 0x5555, 4, 8, O, L * O, colsum=True), buf)


if __name__ == "__main__":
    main()
