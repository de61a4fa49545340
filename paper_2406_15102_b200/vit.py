"""ViT-B/16 for the benchmark workload (BASELINE.json configs[3]).

Written with plain nn.Linear for qkv / proj / fc1 / fc2 / head (torchvision's
vit_b_16 routes attention through nn.MultiheadAttention's packed in_proj, which
a Linear swap would miss -- SURVEY.md 7(vii)) and SDPA for attention.
``convert_linears`` turns every one of those 49 Linear layers into an
HLQLinear; the patch embedding stays a stock Conv2d.
"""
from __future__ import annotations

import torch
import torch.nn as nn
import torch.nn.functional as F


class Block(nn.Module):
    def __init__(self, dim: int, heads: int, mlp: int):
        super().__init__()
        self.heads = heads
        self.ln1 = nn.LayerNorm(dim, eps=1e-6)
        self.qkv = nn.Linear(dim, 3 * dim)
        self.proj = nn.Linear(dim, dim)
        self.ln2 = nn.LayerNorm(dim, eps=1e-6)
        self.fc1 = nn.Linear(dim, mlp)
        self.fc2 = nn.Linear(mlp, dim)

    def forward(self, x):
        B, L, D = x.shape
        # q, k, v as (B, H, L, Dh) views of the qkv output, split along its own
        # (B, L, 3, H, Dh) axis: the backward's stack then writes the qkv
        # gradient (B, L, 3D) contiguously in one copy (the permute(2, 0, 3, 1, 4)
        # form stacked to (3, B, H, L, Dh) and then needed a second, strided copy:
        # ~5 ms per ViT-B/16 step at batch 128 on B200, in both arms)
        q, k, v = self.qkv(self.ln1(x)).view(B, L, 3, self.heads, D // self.heads).unbind(2)
        a = F.scaled_dot_product_attention(q.transpose(1, 2), k.transpose(1, 2), v.transpose(1, 2))
        x = x + self.proj(a.transpose(1, 2).reshape(B, L, D))
        x = x + self.fc2(F.gelu(self.fc1(self.ln2(x))))
        return x


class ViT(nn.Module):
    def __init__(self, image: int = 224, patch: int = 16, dim: int = 768, depth: int = 12,
                 heads: int = 12, mlp: int = 3072, classes: int = 1000):
        super().__init__()
        self.patch = nn.Conv2d(3, dim, patch, stride=patch)
        n = (image // patch) ** 2
        self.cls = nn.Parameter(torch.zeros(1, 1, dim))
        self.pos = nn.Parameter(torch.randn(1, n + 1, dim) * 0.02)
        self.blocks = nn.ModuleList([Block(dim, heads, mlp) for _ in range(depth)])
        self.ln = nn.LayerNorm(dim, eps=1e-6)
        self.head = nn.Linear(dim, classes)

    def forward(self, img):
        x = self.patch(img).flatten(2).transpose(1, 2)
        x = torch.cat([self.cls.expand(x.shape[0], -1, -1), x], dim=1) + self.pos
        for blk in self.blocks:
            x = blk(x)
        return self.head(self.ln(x[:, 0]))


def vit_b16(classes: int = 1000) -> ViT:
    return ViT(classes=classes)


def linear_shapes(batch: int = 128, tokens: int = 197):
    """(name, B, L, I, O) of every Linear in ViT-B/16, one block + the head."""
    return [("qkv", batch, tokens, 768, 2304), ("proj", batch, tokens, 768, 768),
            ("fc1", batch, tokens, 768, 3072), ("fc2", batch, tokens, 3072, 768),
            ("head", batch, 1, 768, 1000)]
