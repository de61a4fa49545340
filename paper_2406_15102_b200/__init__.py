"""B200-native HLQ (Hadamard Low-rank Quantization, arXiv 2406.15102) backward path.

Public names mirror the reference package (/root/reference/pkg/src/hlq/__init__.py)
for the accelerated path; the compute runs in libhlq_b200.so (sm_100a CUDA,
C ABI in include/hlq_b200.h).
"""
from .backprop import (
    ACBPActivation,
    BackwardStrategy,
    GradPair,
    PathSpec,
    QuantizedTensor,
    acbp_compress,
    hlq_backward,
    hlq_grad_weight,
    hq_grad_input,
    ht_axis_for,
    lbp_wht_backward,
    naive_quant_backward,
    strategy_backward,
    vanilla_backward,
)
from .errors import DimensionError, ParameterError, StateError
from .rng import RngState
from .hadamard import DEFAULT_BLOCK, DEFAULT_RANK, HadamardPlan, lowest_sequency_bases, sequency_order

__version__ = "0.1.0"


def __getattr__(name):
    # torch.nn modules are imported lazily so `import paper_2406_15102_b200` stays light
    if name in ("HLQLinear", "HLQLinearFunction", "convert_linears", "refresh_weight_codes"):
        from . import layers
        return getattr(layers, name)
    if name in ("NonFiniteGuard", "check_nonfinite", "install_nonfinite_check"):
        from . import nonfinite
        return getattr(nonfinite, name)
    raise AttributeError(name)
