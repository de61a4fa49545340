"""RngState mirror for true stochastic rounding (reference quantize.py:26-59).

Only the host-side integer bookkeeping lives here -- the 64-bit seed, the
draw counter and the splitmix64 split that gives every quantization site its
own stream (backprop.py:42-43 tags).  The draws themselves are generated on
the GPU (hlq_stochastic.cu reproduces numpy's Philox4x64-10 stream bit for
bit).  Any object with integer ``seed`` / ``counter`` attributes -- e.g. the
reference's own RngState -- is accepted wherever an RngState is.
"""
from __future__ import annotations

from dataclasses import dataclass

_M64 = (1 << 64) - 1
TAG_GX_LEFT, TAG_GX_RIGHT = 11, 12
TAG_GW_LEFT, TAG_GW_RIGHT = 21, 22


def _splitmix64(x: int) -> int:
    x = (x + 0x9E3779B97F4A7C15) & _M64
    x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & _M64
    x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & _M64
    return (x ^ (x >> 31)) & _M64


@dataclass
class RngState:
    """Deterministic, splittable stream: a 64-bit seed plus a draw counter
    (quantize.py:33-46)."""

    seed: int
    counter: int = 0

    def __post_init__(self):
        self.seed = int(self.seed) & _M64

    def split(self, *path: int) -> "RngState":
        """quantize.py:48-52."""
        key = self.seed
        for p in path:
            key = _splitmix64(key ^ _splitmix64(int(p) & _M64))
        return RngState(seed=key)


def site_key(rng, tag: int) -> tuple:
    """(seed, counter) of the Philox key the reference's _quant(.., rng, tag)
    draws with: rng.split(tag) is a fresh state, counter 0 (backprop.py:206-209)."""
    seed = int(getattr(rng, "seed")) & _M64
    child = RngState(seed).split(tag)
    return child.seed, child.counter
