"""B200-native AFMM product (arXiv 1308.2400) behind the reference's hot-path API.

The product path is libafmm_b200.so (include/afmm_b200.h): sm_100a CUDA kernels
with a C ABI. This package is the Python binding of that ABI plus the
synthetic-input generators and the multi-GPU row partition used by bench.py.
"""
from .afmm import (  # noqa: F401
    FAST,
    FAST_LADDER,
    FORM_KERNELS,
    FORMS,
    ORDER_PRESERVING,
    DeviceContext,
    DeviceError,
    DomainError,
    InvalidArgument,
    MultiplyResult,
    OpCounts,
    ShapeError,
    UnsupportedError,
    afmm_case_a,
    afmm_case_b,
    case_a_statistics,
    fp_add_peak,
    generate,
    kernel_launch_count,
    model_partition_case_a,
    model_slab_times_case_a,
    partition_rows,
)

__all__ = [
    "afmm_case_a", "afmm_case_b", "MultiplyResult", "OpCounts", "ShapeError", "DomainError",
    "InvalidArgument", "UnsupportedError", "DeviceError", "DeviceContext", "partition_rows",
    "fp_add_peak", "kernel_launch_count", "ORDER_PRESERVING", "FAST", "FAST_LADDER", "case_a_statistics",
    "model_partition_case_a", "model_slab_times_case_a", "FORMS", "FORM_KERNELS", "generate",
]
