"""paper_2510_19366_b200 -- B200-native (sm_100a) MoE-Prism sub-expert MoE layer.

The product is the C-ABI library ``libmoeprism_b200.so`` (hand-written CUDA
kernels + C++ host code, headers in ``include/moeprism/``).  This package only
binds it (``_lib``), mirrors the C++ host API in Python (``layer``) and runs
the multi-GPU expert-parallel exchange over torch.distributed (``ep``).
"""
from ._lib import CudaError, IoError, ValidationError  # noqa: F401
from .layer import MoeLayer, read_mpex, read_partition_doc, synth_fill, validate_partition  # noqa: F401

__all__ = ["MoeLayer", "synth_fill", "read_mpex", "read_partition_doc", "validate_partition", "ValidationError",
           "IoError", "CudaError"]
