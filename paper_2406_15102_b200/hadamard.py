"""Hadamard plan (host-side configuration only).

Mirrors the configuration surface of the reference's hadamard module
(/root/reference/pkg/src/hlq/hadamard.py:19-106): block size, kept basis
indices (rank r), and the default lowest-sequency basis rule.  The transforms
themselves run on the GPU (csrc/hlq_transform.cu); the kernels receive the
plan as a 16-bit basis bitmap.
"""
from __future__ import annotations

from dataclasses import dataclass, field, replace

from .errors import ParameterError

DEFAULT_BLOCK = 16
DEFAULT_RANK = 8
GPU_BLOCK = 16  # the only block size the sm_100a kernels implement (the HLQ design point)


def sequency_order(block_size: int) -> tuple:
    """Natural-order Walsh rows sorted by sequency, ties toward the lower index
    (hadamard.py:24-43)."""
    if block_size < 2 or block_size & (block_size - 1):
        raise ParameterError(f"block size must be a power of two >= 2, got {block_size}")
    k = block_size.bit_length() - 1

    def seq(i: int) -> int:
        rev = int(format(i, f"0{k}b")[::-1], 2)
        g, s = rev, 1
        while s < 32:
            g ^= g >> s
            s <<= 1
        return g

    return tuple(sorted(range(block_size), key=lambda i: (seq(i), i)))


def lowest_sequency_bases(block_size: int, rank: int) -> tuple:
    return tuple(sorted(sequency_order(block_size)[:rank]))


@dataclass(frozen=True)
class HadamardPlan:
    """Block size, axis and kept bases (hadamard.py:52-106)."""

    block_size: int = DEFAULT_BLOCK
    axis: int = -1
    basis_indices: tuple = field(
        default_factory=lambda: lowest_sequency_bases(DEFAULT_BLOCK, DEFAULT_RANK))

    def __post_init__(self):
        n = self.block_size
        if n < 2 or n & (n - 1):
            raise ParameterError(f"block_size must be a power of two >= 2, got {n}")
        if n > 1024:
            raise ParameterError(f"block_size {n} exceeds the supported maximum 1024")
        idx = tuple(int(i) for i in self.basis_indices)
        if not 1 <= len(idx) <= n:
            raise ParameterError(f"need between 1 and {n} basis indices, got {len(idx)}")
        if len(set(idx)) != len(idx) or list(idx) != sorted(idx):
            raise ParameterError("basis_indices must be distinct and sorted ascending")
        if idx[0] < 0 or idx[-1] >= n:
            raise ParameterError(f"basis indices must lie in [0, {n}), got {idx}")
        object.__setattr__(self, "basis_indices", idx)

    @property
    def rank(self) -> int:
        return len(self.basis_indices)

    @property
    def full_rank(self) -> bool:
        return self.rank == self.block_size

    def with_rank(self, rank: int) -> "HadamardPlan":
        if not 1 <= rank <= self.block_size:
            raise ParameterError(f"rank must be in [1, {self.block_size}], got {rank}")
        return replace(self, basis_indices=lowest_sequency_bases(self.block_size, rank))

    def with_bases(self, basis_indices) -> "HadamardPlan":
        return replace(self, basis_indices=tuple(sorted(int(i) for i in basis_indices)))

    def basis_bitmap(self) -> int:
        bm = 0
        for i in self.basis_indices:
            bm |= 1 << i
        return bm

    @classmethod
    def from_bitmap(cls, block_size: int, bitmap: int, axis: int = -1) -> "HadamardPlan":
        return cls(block_size=block_size, axis=axis,
                   basis_indices=tuple(i for i in range(block_size) if bitmap >> i & 1))

    def gpu_bitmap(self) -> int:
        """The kernels' bitmap; only block 16 has an sm_100a implementation."""
        if self.block_size != GPU_BLOCK:
            raise ParameterError(
                f"the B200 kernels implement block_size {GPU_BLOCK} only, got {self.block_size}")
        return self.basis_bitmap()


def select_bases(means, rank: int) -> tuple:
    """hadamard.py:174-188: the `rank` bases with the largest mean |coefficient|
    (ties toward the lower index), returned ascending.  `means`: 16 values."""
    import numpy as np
    m = np.asarray(means, dtype=np.float64).reshape(-1)
    n = m.size
    if not 1 <= rank <= n:
        raise ParameterError(f"rank must be in [1, {n}], got {rank}")
    order = np.argsort(-m, kind="stable")
    return tuple(sorted(int(i) for i in order[:rank]))
