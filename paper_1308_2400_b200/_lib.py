"""ctypes binding of libafmm_b200.so (the C ABI declared in include/afmm_b200.h).

The library is built in-tree by ``make`` (or ``__graft_entry__.build()``). There
is no fallback: if the shared object is missing or no CUDA device is usable,
the compute entry points fail loudly.
"""
from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, c_char, c_double, c_int32, c_uint32, c_uint64, c_void_p

_HERE = os.path.dirname(os.path.abspath(__file__))
# AFMM_LIB overrides the in-tree library (kernel experiments built under build/).
LIB_PATH = os.environ.get("AFMM_LIB") or os.path.join(_HERE, "libafmm_b200.so")

ABI_VERSION = 2

# afmm_status
OK = 0
ERR_SHAPE = 1
ERR_DOMAIN = 2
ERR_INVALID_ARGUMENT = 3
ERR_CUDA = 4
ERR_UNSUPPORTED = 5
ERR_OUT_OF_MEMORY = 6

CASE_A = 0
CASE_B = 1
F64 = 0
F32 = 1
MODE_ORDER_PRESERVING = 0
MODE_FAST = 1
MODE_FAST_LADDER = 2

# afmm_error_kind
ERRKIND_NONE = 0
ERRKIND_NOT_INTEGER = 1
ERRKIND_OUT_OF_RANGE = 2
ERRKIND_NON_FINITE = 3
ERRKIND_SHAPE = 4
ERRKIND_EMPTY = 5
ERRKIND_REP_TOO_LARGE = 6  # unused since ABI 2
ERRKIND_REP_NAN = 8
ERRKIND_OTHER = 7


class OpCounts(ctypes.Structure):
    """op_counts.hpp:17-23"""

    _fields_ = [("additions", c_uint64), ("multiplications", c_uint64), ("zero_skips", c_uint64)]

    def as_tuple(self):
        return (int(self.additions), int(self.multiplications), int(self.zero_skips))


class Error(ctypes.Structure):
    _fields_ = [
        ("kind", c_int32),
        ("operand", c_int32),
        ("row", c_uint64),
        ("col", c_uint64),
        ("value", c_double),
        ("message", c_char * 256),
    ]


class IpcHandle(ctypes.Structure):
    _fields_ = [("bytes", ctypes.c_uint8 * 64), ("offset", c_uint64)]


class Timing(ctypes.Structure):
    """afmm_timing: device-measured phases of one host-buffer call."""

    _fields_ = [("total_ms", ctypes.c_float), ("compute_ms", ctypes.c_float),
                ("devices", c_int32), ("form", c_int32)]


PARTITION_WORK = 0
PARTITION_ROWS = 1


class Options(ctypes.Structure):
    """afmm_options (ABI 2)."""

    _fields_ = [("mode", c_int32), ("device", c_int32), ("split_k", c_int32),
                ("num_devices", c_int32), ("devices", POINTER(c_int32)), ("partition", c_int32),
                ("flags", c_int32), ("timing", POINTER(Timing))]


FLAG_KERNEL_SEMANTICS = 1

ROLE_REAL = 0
ROLE_INTEGER = 1


class GeneratorSpec(ctypes.Structure):
    """afmm_generator_spec: the reference's GeneratorSpec (random.hpp:30-58)."""

    _fields_ = [("n", c_uint64), ("density", c_double), ("mu_prime", c_double),
                ("role", c_int32), ("value_low", c_double), ("value_high", c_double)]


# Every symbol include/afmm_b200.h declares, with its ctypes signature.
_SIGNATURES = {
    "afmm_case_a_f64": (c_int32, [c_void_p, c_uint64, c_void_p, c_uint64, c_void_p,
                                  POINTER(Options), POINTER(OpCounts), POINTER(Error)]),
    "afmm_case_b_f64": (c_int32, [c_void_p, c_uint64, c_void_p, c_uint64, c_void_p,
                                  POINTER(Options), POINTER(OpCounts), POINTER(Error)]),
    "afmm_case_a_f32": (c_int32, [c_void_p, c_uint64, c_void_p, c_uint64, c_void_p,
                                  POINTER(Options), POINTER(OpCounts), POINTER(Error)]),
    "afmm_case_b_f32": (c_int32, [c_void_p, c_uint64, c_void_p, c_uint64, c_void_p,
                                  POINTER(Options), POINTER(OpCounts), POINTER(Error)]),
    "afmm_context_create": (c_int32, [c_int32, POINTER(c_void_p)]),
    "afmm_context_destroy": (None, [c_void_p]),
    "afmm_context_set_stream": (c_int32, [c_void_p, c_void_p]),
    "afmm_product_device": (c_int32, [c_void_p, c_int32, c_int32, c_void_p, c_void_p, c_uint64,
                                      c_uint64, c_void_p, c_uint64, c_uint64, c_uint64,
                                      POINTER(Options), c_int32, POINTER(OpCounts),
                                      POINTER(Error)]),
    "afmm_context_finish": (c_int32, [c_void_p, POINTER(OpCounts), POINTER(Error)]),
    "afmm_context_enable_timing": (c_int32, [c_void_p, c_int32]),
    "afmm_context_last_timing": (c_int32, [c_void_p, POINTER(ctypes.c_float),
                                           POINTER(ctypes.c_float), POINTER(ctypes.c_float)]),
    "afmm_context_last_form": (c_int32, [c_void_p]),
    "afmm_row_work_device": (c_int32, [c_void_p, c_int32, c_int32, c_void_p, c_void_p, c_uint64,
                                       c_uint64, POINTER(c_uint64), POINTER(Error)]),
    "afmm_row_cost_device": (c_int32, [c_void_p, c_int32, c_int32, c_void_p, c_void_p, c_uint64,
                                       c_uint64, POINTER(c_uint64), POINTER(Error)]),
    "afmm_partition_device": (c_int32, [c_void_p, c_int32, c_int32, c_void_p, c_void_p, c_uint64,
                                        c_uint64, c_uint32, POINTER(c_uint64), POINTER(Error)]),
    "afmm_model_partition_case_a": (c_int32, [c_int32, c_uint64, c_int32, POINTER(c_uint64),
                                              POINTER(c_uint32), c_uint32, POINTER(c_uint64),
                                              POINTER(c_double)]),
    "afmm_model_slab_time_case_a": (c_int32, [c_int32, c_uint64, c_int32, POINTER(c_uint64),
                                              POINTER(c_uint32), c_uint64, c_uint64,
                                              POINTER(c_double)]),
    "afmm_partition_rows": (c_int32, [POINTER(c_uint64), c_uint64, c_uint32, POINTER(c_uint64)]),
    "afmm_fp_add_peak": (c_int32, [c_int32, c_int32, POINTER(c_double), POINTER(c_double)]),
    "afmm_generate_f64": (c_int32, [POINTER(GeneratorSpec), c_uint64, c_void_p, POINTER(Options),
                                    POINTER(Error)]),
    "afmm_generate_f32": (c_int32, [POINTER(GeneratorSpec), c_uint64, c_void_p, POINTER(Options),
                                    POINTER(Error)]),
    "afmm_generate_device": (c_int32, [c_void_p, POINTER(GeneratorSpec), c_uint64, c_int32,
                                       c_void_p, c_uint64, POINTER(Error)]),
    "afmm_ipc_export": (c_int32, [c_void_p, POINTER(IpcHandle), POINTER(Error)]),
    "afmm_ipc_open": (c_int32, [c_int32, POINTER(IpcHandle), POINTER(c_void_p), POINTER(Error)]),
    "afmm_ipc_close": (c_int32, [c_void_p]),
    "afmm_kernel_launch_count": (c_uint64, []),
    "afmm_status_string": (ctypes.c_char_p, [c_int32]),
    "afmm_abi_version": (c_int32, []),
}

EXPORTED_SYMBOLS = tuple(_SIGNATURES)

_lib = None


def load() -> ctypes.CDLL:
    """Load libafmm_b200.so (once). Raises RuntimeError if it was not built."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(
            f"libafmm_b200.so not found at {LIB_PATH}: build it with `make` or "
            "`python -c 'import __graft_entry__ as g; g.build()'` (there is no CPU fallback)")
    lib = ctypes.CDLL(LIB_PATH)
    if lib.afmm_abi_version() != ABI_VERSION:
        raise RuntimeError(f"{LIB_PATH}: ABI {lib.afmm_abi_version()}, this binding expects "
                           f"{ABI_VERSION} (rebuild with `make`)")
    for name, (res, args) in _SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def status_string(code: int) -> str:
    return load().afmm_status_string(code).decode()
