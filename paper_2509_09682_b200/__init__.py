"""B200-native (sm_100a) Cut Cross-Entropy and CCE- loss path.

Drop-in for the lseforge loss entry points (cce_forward / cce_backward /
ccem_forward / ccem_backward / ccem_backward_rows / estimate_flops, with the
CceConfig::filter_eps gradient filter).  Compute runs in liblseforge_b200.so
(hand-written CUDA for sm_100a behind the C-ABI in include/lseforge_b200.h);
this package is the host-side mirror of the reference interface.
"""
from . import _capi
from .accountant import MemAccountant, Report, ScalarKind
from .cce import (CceBackwardResult, CceConfig, cce_backward, cce_forward, cce_forward_backward,
                  kFp16MinPositive)
from .ccem import (Backend, FlopEstimate, backend_is_sampled, ccem_backward, ccem_backward_rows,
                   ccem_forward_backward,
                   ccem_forward, estimate_flops)
from .losses import (GradPair, LossOutput, ce_full_backward, ce_full_forward, ce_sampled_backward,
                     ce_sampled_forward, validate_loss_inputs)
from .adam import AdamConfig, DeviceAdam
from .metrics import EvalSummary, evaluate
from .sampler import sample_popularity, sample_uniform

__all__ = [
    "CceConfig", "CceBackwardResult", "cce_forward", "cce_backward", "cce_forward_backward",
    "kFp16MinPositive",
    "ccem_forward", "ccem_backward", "ccem_backward_rows", "ccem_forward_backward", "estimate_flops",
    "FlopEstimate",
    "Backend", "backend_is_sampled", "LossOutput", "GradPair", "validate_loss_inputs",
    "MemAccountant", "Report", "ScalarKind", "sample_uniform", "sample_popularity", "ce_full_forward",
    "ce_full_backward", "EvalSummary", "evaluate", "AdamConfig", "DeviceAdam", "lib",
]


def lib():
    """The loaded liblseforge_b200.so (raises if it has not been built)."""
    return _capi.lib()
