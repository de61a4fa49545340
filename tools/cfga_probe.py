import sys, json, torch
sys.path.insert(0, ".")
from paper_2406_15102_b200 import ops
from tools.stage_bench import timeit
flush = torch.empty(64 * 1024 * 1024, device="cuda")
T, I, O = 4096, 1024, 1024
x = torch.randn(T, I, device="cuda"); w = torch.randn(O, I, device="cuda") * 0.04
gy = torch.randn(T, O, device="cuda") * 1e-3
cw, _, sw, _ = ops.quant_proj_rows(w, 1, O, I, 0xFFFF, 4)
res = {}
for bm in (0x0101, 0x5555):
    xp, k, sx, _ = ops.quant_proj_rows(x, 1, T, I, bm, 8)
    cgx, sgx, cg, kg, sg, _ = ops.quant_dual(gy, 1, T, O, bm, 4, 8)
    r = {}
    r["dual"] = timeit(lambda: ops.quant_dual(gy, 1, T, O, bm, 4, 8), flush=flush)
    r["dw"] = timeit(lambda: ops.gemm_i8(cg, xp, O, I, k, 8, 8, sg, sx, 1.0, exact=False), flush=flush)
    r["dx"] = timeit(lambda: ops.gemm_i8(cgx, cw, T, I, ops.pad16(O), 4, 4, sgx, sw, 1.0, exact=False), flush=flush)
    r["pair"] = timeit(lambda: ops.gemm_i8_pair(dict(a=cg, b=xp, m=O, n=I, k=k, bits_a=8, bits_b=8, sa=sg, sb=sx),
                             dict(a=cgx, b=cw, m=T, n=I, k=ops.pad16(O), bits_a=4, bits_b=4, sa=sgx, sb=sw)), flush=flush)
    xb, gb, wb = x.bfloat16(), gy.bfloat16(), w.bfloat16()
    r["torch_int_mm_dx"] = timeit(lambda: torch._int_mm(cgx, cw.t()), flush=flush)
    r["dense_dx"] = timeit(lambda: gb @ wb, flush=flush)
    r["dense_dw"] = timeit(lambda: gb.t() @ xb, flush=flush)
    res[f"r{bin(bm).count('1')}_K{k}"] = {a: round(b, 1) for a, b in r.items()}
print(json.dumps(res))
