"""Lazy non-finite detection for the HLQ training path.

The reference refuses to quantize NaN / Inf (``ValueError("cannot quantize
non-finite values")``, quantize.py:119-120,138-139; tensor.py:36-37).  Checking
every operand on the host would cost one synchronisation per layer.  Instead
every transform kernel ORs its operand's non-finite status (amax bits >=
0x7F800000, which NaN / Inf inputs always produce) into a per-device sticky
word, and the caller checks it when it chooses -- typically once per step,
before the optimizer applies the gradients:

    guard = install_nonfinite_check(optimizer)   # raises ValueError in optimizer.step()

``NonFiniteGuard.fetch()`` only enqueues a 4-byte copy (and reset) on the
current stream into pinned host memory, so it can run ahead of the host;
``check()`` waits for that copy and raises.
"""
from __future__ import annotations

import torch

from . import _lib, ops


class NonFiniteGuard:
    def __init__(self, device=None):
        self.device = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
        self.host = torch.zeros(1, dtype=torch.int32).pin_memory()
        self.event = None

    def fetch(self, reset: bool = True) -> None:
        """Enqueue copy (+ reset) of the device's flag; no host synchronisation."""
        with torch.cuda.device(self.device):
            _lib.call("hlq_nonfinite_fetch", ops._p(self.host), int(reset), ops._stream())
            self.event = torch.cuda.Event()
            self.event.record()

    def check(self) -> None:
        """Raise ValueError if any HLQ operand since the last reset held NaN / Inf."""
        if self.event is None:
            self.fetch()
        self.event.synchronize()
        self.event = None
        if int(self.host[0]) != 0:
            raise ValueError("cannot quantize non-finite values (an HLQ backward operand held NaN/Inf)")


def check_nonfinite(device=None) -> None:
    """Fetch, reset and check the flag now (one host synchronisation)."""
    NonFiniteGuard(device).check()


def install_nonfinite_check(optimizer: torch.optim.Optimizer, device=None) -> NonFiniteGuard:
    """Check the flag in a step pre-hook: optimizer.step() raises ValueError
    (before touching the parameters) when the backward saw NaN / Inf."""
    guard = NonFiniteGuard(device)
    optimizer.register_step_pre_hook(lambda opt, args, kwargs: guard.check())
    return guard
