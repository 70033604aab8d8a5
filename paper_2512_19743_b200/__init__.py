"""B200-native sparse APML (CUDA-APML, arXiv 2512.19743): C-ABI libapml.so + thin binding.

The hot path lives in csrc/ (sm_100a CUDA) behind include/apml.h.  This package never
imports the test oracle and has no CPU fallback.
"""
from .apml import Config, Context, Plan, apml_loss, forward, loss_grad_host  # noqa: F401

__all__ = ["Config", "Context", "Plan", "apml_loss", "forward", "loss_grad_host"]
