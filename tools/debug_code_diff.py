import sys, numpy as np, torch
sys.path.insert(0, '.')
from oracle import hlq_oracle as orc
import paper_2406_15102_b200 as h
from paper_2406_15102_b200 import ops
name, I, O = "qkv", 768, 2304
B, L = 128, 197
x, w, gy = orc.make_inputs(len(name) * 31 + O, (B, L, I), (O, I), (B, L, O))
g = torch.from_numpy(gy).cuda()
for variant in ("ht_cols", "dual"):
    if variant == "ht_cols":
        c, s, _ = ops.quant_ht_cols(g.reshape(B * L, O), 4)
    else:
        c, s, *_ = ops.quant_dual(g, B, L, O, 0x5555, 4, 8, O, L * O)
    c = c[:, :O].cpu().numpy()
    v = orc.transform_axis(gy, 2, 16).reshape(B * L, -1)
    ref, rs = orc.quantize(v, 4)
    d = np.argwhere(c != ref)
    print(variant, "scale", float(s.cpu()[0]), float(rs), "ndiff", len(d))
    for r, col in d[:5]:
        vv = np.float32(v[r, col])
        q = vv / rs
        print(" at", r, col, "v", repr(vv), hex(vv.view(np.uint32)), "q", repr(q), "floor", np.floor(q),
              "frac*2048", (q - np.floor(q)) * np.float32(2048), "u", vv.view(np.uint32) & 0x7FF,
              "ours", c[r, col], "ref", ref[r, col])
        print("   block inputs", gy.reshape(B * L, O)[r, (col // 16) * 16:(col // 16) * 16 + 16])
