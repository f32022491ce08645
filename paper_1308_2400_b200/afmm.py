"""Python mirror of the reference's AFMM hot-path API, backed by the sm_100a C ABI.

Reference interface (paths relative to /root/reference/proj):
  afmm::afmm_case_a(const DenseMatrix& lhs, const DenseMatrix& rhs) -> MultiplyResult
      include/afmm/kernels.hpp:113-136  (real lhs bases, integer rhs reps)
  afmm::afmm_case_b(...)               include/afmm/kernels.hpp:142-165
  OpCounts / MultiplyResult            include/afmm/op_counts.hpp:17-33
  shape_error                          include/afmm/errors.hpp:9-12

Same names, same argument meaning, same error behaviour: a dimension mismatch
raises ShapeError (a ValueError, as shape_error is a std::invalid_argument),
a non-integer or out-of-range rep raises DomainError naming the first
offender in row-major order with the reference's message text, an empty
matrix raises InvalidArgument ("DenseMatrix: dimension must be >= 1").

Every product is computed by the CUDA kernels in csrc/ through
libafmm_b200.so; nothing here computes on the CPU.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass
from typing import Optional, Sequence, Tuple

import numpy as np

from . import _lib

ORDER_PRESERVING = "order-preserving"
FAST = "fast"
FAST_LADDER = "fast-ladder"  # fast + each term's |rep| copies summed as a doubling ladder
_MODES = {ORDER_PRESERVING: _lib.MODE_ORDER_PRESERVING, FAST: _lib.MODE_FAST,
          FAST_LADDER: _lib.MODE_FAST_LADDER}


class ShapeError(ValueError):
    """afmm::shape_error (errors.hpp:9-12): dimension mismatch."""


class DomainError(ValueError):
    """std::domain_error: rep not integer-valued / out of range / non-finite element."""


class InvalidArgument(ValueError):
    """std::invalid_argument: empty matrix or invalid option."""


class UnsupportedError(InvalidArgument):
    """n beyond the device index range (2^31 - 1). (Every rep the reference
    accepts, |rep| <= 2^53, is accepted: a rep beyond one list entry's range is
    split into consecutive entries at the same k.)"""


class DeviceError(RuntimeError):
    """CUDA failure or no usable device (there is no CPU fallback)."""


@dataclass(frozen=True)
class OpCounts:
    """op_counts.hpp:17-23"""

    additions: int = 0
    multiplications: int = 0
    zero_skips: int = 0


@dataclass
class MultiplyResult:
    """op_counts.hpp:30-33 (+ the device timing of the call when requested)"""

    product: np.ndarray
    counts: OpCounts
    timing: Optional[dict] = None


def _raise_for(status: int, err: _lib.Error) -> None:
    if status == _lib.OK:
        return
    msg = err.message.decode(errors="replace") or _lib.status_string(status)
    if status == _lib.ERR_SHAPE:
        raise ShapeError(msg)
    if status == _lib.ERR_DOMAIN:
        raise DomainError(msg)
    if status == _lib.ERR_UNSUPPORTED:
        raise UnsupportedError(msg)
    if status == _lib.ERR_INVALID_ARGUMENT:
        raise InvalidArgument(msg)
    if status == _lib.ERR_OUT_OF_MEMORY:
        raise MemoryError(msg)
    raise DeviceError(msg)


_PARTITIONS = {"work": _lib.PARTITION_WORK, "rows": _lib.PARTITION_ROWS}


def _options(mode: str, device: Optional[int], devices: Optional[Sequence[int]] = None,
             partition: str = "work", split_k: int = 0,
             timing: Optional[_lib.Timing] = None,
             kernel_semantics: bool = False) -> Tuple[_lib.Options, object]:
    """afmm_options + the ctypes objects it points to (kept alive by the caller)."""
    if mode not in _MODES:
        raise InvalidArgument(f"afmm: unknown mode {mode!r}")
    if partition not in _PARTITIONS:
        raise InvalidArgument(f"afmm: unknown partition {partition!r}")
    o = _lib.Options()
    o.mode = _MODES[mode]
    o.device = -1 if device is None else int(device)
    o.split_k = int(split_k)
    o.partition = _PARTITIONS[partition]
    o.flags = _lib.FLAG_KERNEL_SEMANTICS if kernel_semantics else 0
    keep = None
    if devices is not None:
        devs = [int(d) for d in devices]
        if not devs:
            raise InvalidArgument("afmm: devices must not be empty")
        keep = (ctypes.c_int32 * len(devs))(*devs)
        o.num_devices = len(devs)
        o.devices = ctypes.cast(keep, ctypes.POINTER(ctypes.c_int32))
    if timing is not None:
        o.timing = ctypes.pointer(timing)
    return o, keep


def _as_square(m, name: str) -> np.ndarray:
    a = np.asarray(m)
    if a.ndim != 2 or a.shape[0] != a.shape[1]:
        raise ShapeError(f"DenseMatrix: {name} must be square n x n, got shape {a.shape}")
    return a


def _common_dtype(lhs: np.ndarray, rhs: np.ndarray, dtype) -> np.dtype:
    if dtype is not None:
        dt = np.dtype(dtype)
    elif lhs.dtype == np.float32 and rhs.dtype == np.float32:
        dt = np.dtype(np.float32)
    else:
        dt = np.dtype(np.float64)
    if dt not in (np.dtype(np.float32), np.dtype(np.float64)):
        raise InvalidArgument(f"afmm: dtype must be float32 or float64, got {dt}")
    return dt


def _product(which: int, lhs, rhs, mode: str, device: Optional[int], dtype,
             out: Optional[np.ndarray], devices=None, partition: str = "work",
             split_k: int = 0, timing: bool = False,
             kernel_semantics: bool = False) -> MultiplyResult:
    lib = _lib.load()
    l = _as_square(lhs, "lhs")
    r = _as_square(rhs, "rhs")
    dt = _common_dtype(l, r, dtype)
    l = np.ascontiguousarray(l, dtype=dt)
    r = np.ascontiguousarray(r, dtype=dt)
    n = l.shape[0]
    if out is None:
        out = np.empty((n, n), dtype=dt)
    elif out.dtype != dt or out.shape != (n, n) or not out.flags.c_contiguous:
        raise InvalidArgument("afmm: out must be a C-contiguous n x n array of the operand dtype")
    counts = _lib.OpCounts()
    err = _lib.Error()
    tm = _lib.Timing() if timing else None
    opts, _keep = _options(mode, device, devices, partition, split_k, tm, kernel_semantics)
    fn = {
        (_lib.CASE_A, np.float64): lib.afmm_case_a_f64,
        (_lib.CASE_B, np.float64): lib.afmm_case_b_f64,
        (_lib.CASE_A, np.float32): lib.afmm_case_a_f32,
        (_lib.CASE_B, np.float32): lib.afmm_case_b_f32,
    }[(which, dt.type)]
    status = fn(l.ctypes.data, l.shape[0], r.ctypes.data, r.shape[0], out.ctypes.data,
                ctypes.byref(opts), ctypes.byref(counts), ctypes.byref(err))
    _raise_for(status, err)
    t = None
    if tm is not None:
        t = {"total_ms": tm.total_ms, "compute_ms": tm.compute_ms, "devices": tm.devices,
             "form": FORMS.get(tm.form, "bform")}
    return MultiplyResult(out, OpCounts(*counts.as_tuple()), t)


def afmm_case_a(lhs, rhs, *, mode: str = ORDER_PRESERVING, device: Optional[int] = None,
                dtype=None, out: Optional[np.ndarray] = None, devices=None,
                partition: str = "work", split_k: int = 0, timing: bool = False,
                kernel_semantics: bool = False) -> MultiplyResult:
    """AFMM Case A on the GPU: real lhs bases, integer-valued rhs reps (kernels.hpp:113-136).

    devices=[d0, d1, ...] shards the rows of Z over several GPUs in this
    process (a device may repeat); partition="work" balances predicted kernel
    time, "rows" cuts equal row counts. timing=True adds the device-measured
    phases of the call to the result. By default the arrays are the values a
    DenseMatrix is constructed from (a non-finite element is the constructor's
    error, matrix.hpp:31-35); kernel_semantics=True applies only the kernel's
    own checks, as for matrices built element by element (non-finite bases
    are computed, an infinite rep is out of range, a NaN rep unsupported)."""
    return _product(_lib.CASE_A, lhs, rhs, mode, device, dtype, out, devices, partition, split_k,
                    timing, kernel_semantics)


def afmm_case_b(lhs, rhs, *, mode: str = ORDER_PRESERVING, device: Optional[int] = None,
                dtype=None, out: Optional[np.ndarray] = None, devices=None,
                partition: str = "work", split_k: int = 0, timing: bool = False,
                kernel_semantics: bool = False) -> MultiplyResult:
    """AFMM Case B on the GPU: integer-valued lhs reps, real rhs bases (kernels.hpp:142-165).
    Multi-GPU, timing and kernel_semantics options as in afmm_case_a."""
    return _product(_lib.CASE_B, lhs, rhs, mode, device, dtype, out, devices, partition, split_k,
                    timing, kernel_semantics)


# ---- device-resident API ------------------------------------------------------

_DT_CODE = {"float64": _lib.F64, "float32": _lib.F32}


class RawRows:
    """Row-major device rows addressed by a raw pointer (e.g. another GPU's
    buffer opened with ipc_open): usable as `out` of DeviceContext.product."""

    def __init__(self, ptr: int, ld: int, dtype: str, ncols: int, nrows: Optional[int] = None):
        self.ptr, self.ld, self.dtype, self.ncols = int(ptr), int(ld), dtype, int(ncols)
        self.nrows = nrows  # None: unknown (the caller vouches for the extent)

    def rows(self, r0: int) -> "RawRows":
        """The view starting at row r0."""
        es = 4 if self.dtype == "float32" else 8
        return RawRows(self.ptr + r0 * self.ld * es, self.ld, self.dtype, self.ncols,
                       None if self.nrows is None else self.nrows - r0)


def _tensor_info(t, device: Optional[int] = None, what: str = "operand") -> Tuple[int, int, str, int]:
    """(data_ptr, leading dimension, dtype name, ncols) of a 2D row-major CUDA
    tensor on `device` (or a RawRows view)."""
    if isinstance(t, RawRows):
        return t.ptr, t.ld, t.dtype, t.ncols
    if not getattr(t, "is_cuda", False):
        raise InvalidArgument(f"afmm: {what} must be a CUDA tensor (device-resident API)")
    if device is not None and t.device.index != device:
        raise InvalidArgument(f"afmm: {what} is on cuda:{t.device.index}, the context on "
                              f"cuda:{device}")
    if t.dim() != 2 or t.stride(1) != 1:
        raise InvalidArgument("afmm: device operands must be 2D with unit column stride")
    name = str(t.dtype).replace("torch.", "")
    if name not in _DT_CODE:
        raise InvalidArgument(f"afmm: unsupported dtype {t.dtype}")
    return t.data_ptr(), t.stride(0), name, t.shape[1]


# afmm_context_last_form codes (include/afmm_b200.h)
FORMS = {0: "bform", 1: "aform", 2: "split", 4: "group", 6: "split-group"}
# the repeated-addition kernel(s) behind each form (bench lines, profiles)
FORM_KERNELS = {"bform": "k_bform", "aform": "k_aform", "split": "k_aform+k_bform",
                "group": "k_bgroup", "split-group": "k_aform+k_bgroup"}


class DeviceContext:
    """An afmm_context: device, stream binding and grow-only workspace."""

    def __init__(self, device: int = 0):
        self._lib = _lib.load()
        h = ctypes.c_void_p()
        status = self._lib.afmm_context_create(int(device), ctypes.byref(h))
        if status != _lib.OK:
            raise DeviceError(f"afmm_context_create({device}) failed: "
                              f"{_lib.status_string(status)}")
        self._h = h
        self.device = int(device)

    def close(self) -> None:
        if getattr(self, "_h", None):
            self._lib.afmm_context_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_stream(self, stream) -> None:
        """Bind the context to a CUDA stream (a torch.cuda.Stream or a raw
        handle); until then every call runs on torch's current stream."""
        handle = getattr(stream, "cuda_stream", stream)
        self._bind(int(handle or 0))
        self._explicit_stream = True

    def _bind(self, handle: int) -> None:
        if handle != getattr(self, "_bound", None):
            st = self._lib.afmm_context_set_stream(self._h, ctypes.c_void_p(handle))
            if st != _lib.OK:
                raise DeviceError(f"afmm_context_set_stream: {_lib.status_string(st)}")
            self._bound = handle

    def _follow_torch_stream(self) -> None:
        if not getattr(self, "_explicit_stream", False):
            import torch

            self._bind(int(torch.cuda.current_stream(self.device).cuda_stream))

    def generate(self, out, density: float, mu_prime: float, integer: bool, seed: int,
                 low: float = 0.5, high: float = 1.5) -> None:
        """afmm::generate (random.hpp:111-129) on this context's device, into the
        n x n device tensor `out` (float64, or float32 = the values rounded):
        operands for `product` without a host round trip."""
        p, ld, dname, n = _tensor_info(out, self.device, "out")
        if out.shape[0] != n:
            raise InvalidArgument("afmm: out must be n x n")
        spec = _gen_spec(n, density, mu_prime, integer, low, high)
        err = _lib.Error()
        status = self._lib.afmm_generate_device(self._h, ctypes.byref(spec),
                                                int(seed) & 0xFFFFFFFFFFFFFFFF, _DT_CODE[dname],
                                                p, ld, ctypes.byref(err))
        _raise_for(status, err)

    def product(self, which: str, lhs, rhs, out, row_begin: int = 0,
                row_end: Optional[int] = None, *, sync: bool = True,
                mode: str = ORDER_PRESERVING, split_k: int = 0) -> Optional[OpCounts]:
        """Rows [row_begin, row_end) of Z into `out` (device tensors on this
        context's device, row-major; `out` row r holds Z row row_begin + r)."""
        lp, ld, dname, n = _tensor_info(lhs, self.device, "lhs")
        rp, ld_r, dname_r, n_r = _tensor_info(rhs, self.device, "rhs")
        if dname_r != dname or ld_r != ld or lhs.shape[0] != n or rhs.shape != lhs.shape:
            raise ShapeError(f"afmm_case_{which}: dimension mismatch {n} vs {n_r}")
        row_end = n if row_end is None else int(row_end)
        row_begin = int(row_begin)
        if not 0 <= row_begin <= row_end <= n:
            raise InvalidArgument(f"afmm: rows [{row_begin}, {row_end}) outside [0, {n})")
        op, ld_out, dname_o, ncols_o = _tensor_info(out, self.device, "out")
        if dname_o != dname:
            raise InvalidArgument("afmm: out dtype differs from the operands")
        rows_o = out.nrows if isinstance(out, RawRows) else out.shape[0]
        if row_end > row_begin and (ncols_o < n or (rows_o is not None and
                                                    rows_o < row_end - row_begin)):
            raise InvalidArgument(f"afmm: out holds {rows_o} x {ncols_o}, the slab needs "
                                  f"{row_end - row_begin} x {n}")
        self._follow_torch_stream()
        counts = _lib.OpCounts()
        err = _lib.Error()
        opts, _ = _options(mode, self.device, split_k=split_k)
        status = self._lib.afmm_product_device(
            self._h, _lib.CASE_A if which == "a" else _lib.CASE_B, _DT_CODE[dname], lp, rp, n, ld,
            op, ld_out, row_begin, row_end, ctypes.byref(opts), 1 if sync else 0,
            ctypes.byref(counts), ctypes.byref(err))
        _raise_for(status, err)
        return OpCounts(*counts.as_tuple()) if sync else None

    def enable_timing(self, enable: bool = True) -> None:
        self._lib.afmm_context_enable_timing(self._h, 1 if enable else 0)

    def last_timing(self) -> Tuple[float, float, float]:
        """(prepass, repeated-addition kernel, epilogue) milliseconds of the last product."""
        v = [ctypes.c_float() for _ in range(3)]
        self._lib.afmm_context_last_timing(self._h, *[ctypes.byref(x) for x in v])
        return tuple(x.value for x in v)

    def last_form(self) -> str:
        """Kernel(s) of the last product: "bform" (rep uniform per warp), "aform"
        (Case A, base uniform per warp), "split" (Case A rows divided between
        the two), "group" / "split-group" (the B-form part ran the small-rep
        group kernel k_bgroup: fp32, every rep in 0..2)."""
        return FORMS.get(self._lib.afmm_context_last_form(self._h), "bform")

    def finish(self) -> OpCounts:
        counts = _lib.OpCounts()
        err = _lib.Error()
        _raise_for(self._lib.afmm_context_finish(self._h, ctypes.byref(counts), ctypes.byref(err)),
                   err)
        return OpCounts(*counts.as_tuple())

    def _row_query(self, fn, which: str, lhs, rhs) -> np.ndarray:
        lp, ld, dname, n = _tensor_info(lhs, self.device, "lhs")
        rp, _, _, _ = _tensor_info(rhs, self.device, "rhs")
        self._follow_torch_stream()
        out = np.zeros(n, dtype=np.uint64)
        err = _lib.Error()
        status = fn(self._h, _lib.CASE_A if which == "a" else _lib.CASE_B, _DT_CODE[dname], lp, rp,
                    n, ld, out.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)), ctypes.byref(err))
        _raise_for(status, err)
        return out

    def row_work(self, which: str, lhs, rhs) -> np.ndarray:
        """W_i: exact additions of each Z row (afmm_row_work_device)."""
        return self._row_query(self._lib.afmm_row_work_device, which, lhs, rhs)

    def partition(self, which: str, lhs, rhs, parts: int) -> np.ndarray:
        """Row cuts for `parts` devices (afmm_partition_device): equal W_i for
        Case B, equal modeled kernel time for Case A."""
        lp, ld, dname, n = _tensor_info(lhs, self.device, "lhs")
        rp, _, _, _ = _tensor_info(rhs, self.device, "rhs")
        self._follow_torch_stream()
        cuts = np.zeros(int(parts) + 1, dtype=np.uint64)
        err = _lib.Error()
        status = self._lib.afmm_partition_device(
            self._h, _lib.CASE_A if which == "a" else _lib.CASE_B, _DT_CODE[dname], lp, rp, n, ld,
            int(parts), cuts.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)), ctypes.byref(err))
        _raise_for(status, err)
        return cuts.astype(np.int64)

    def row_cost(self, which: str, lhs, rhs) -> np.ndarray:
        """Predicted kernel time of each Z row (afmm_row_cost_device): W_i for
        Case B, the Case A cost model (cheaper of A-form and B-form) for Case A."""
        return self._row_query(self._lib.afmm_row_cost_device, which, lhs, rhs)


def partition_rows(work, parts: int) -> np.ndarray:
    """Contiguous row ranges of near-equal total work (afmm_partition_rows)."""
    lib = _lib.load()
    w = np.ascontiguousarray(work, dtype=np.uint64)
    cuts = np.zeros(int(parts) + 1, dtype=np.uint64)
    status = lib.afmm_partition_rows(w.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)), w.size,
                                     int(parts), cuts.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)))
    if status != _lib.OK:
        raise InvalidArgument("afmm_partition_rows: invalid arguments")
    return cuts.astype(np.int64)


def case_a_statistics(lhs: np.ndarray, rhs: np.ndarray):
    """(stats[4], nnz_row[n]) of a Case A problem as the prepass computes them
    (host restatement for model queries): nonzero reps of Y, sum over (k,
    A-form tile) of the tile's max |rep|, reps beyond 2048, sum of |rep|; and
    the nonzero bases of each row of X."""
    n = lhs.shape[0]
    tile = 1024 if lhs.dtype == np.float32 else 512
    reps = np.where(rhs != 0, np.rint(rhs.astype(np.float64)), 0).astype(np.int64)
    # llround rounds half away from zero; np.rint to even: fix the halves
    half = np.abs(rhs.astype(np.float64) - np.trunc(rhs.astype(np.float64))) == 0.5
    reps[half] = (np.trunc(rhs[half]) + np.sign(rhs[half])).astype(np.int64)
    a = np.abs(reps)
    ntiles = (n + tile - 1) // tile
    trip = 0
    for t in range(ntiles):
        trip += int(np.minimum(a[:, t * tile:(t + 1) * tile], 2048).max(axis=1).sum())
    stats = np.array([int((a != 0).sum()), trip, int((a > 2048).sum()), int(a.sum())],
                     dtype=np.uint64)
    nnz_row = (lhs != 0).sum(axis=1).astype(np.uint32)
    return stats, nnz_row


def model_partition_case_a(stats, nnz_row, parts: int, dtype: str = "float32",
                           sms: int = 148) -> Tuple[np.ndarray, np.ndarray]:
    """Case A row cuts by modeled kernel time and each slab's modeled cycles
    (afmm_model_partition_case_a; host only, no device)."""
    lib = _lib.load()
    st = np.ascontiguousarray(stats, dtype=np.uint64)
    nz = np.ascontiguousarray(nnz_row, dtype=np.uint32)
    cuts = np.zeros(int(parts) + 1, dtype=np.uint64)
    cyc = np.zeros(int(parts), dtype=np.float64)
    status = lib.afmm_model_partition_case_a(
        _DT_CODE[dtype], nz.size, int(sms), st.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)),
        nz.ctypes.data_as(ctypes.POINTER(ctypes.c_uint32)), int(parts),
        cuts.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)),
        cyc.ctypes.data_as(ctypes.POINTER(ctypes.c_double)))
    if status != _lib.OK:
        raise InvalidArgument("afmm_model_partition_case_a: invalid arguments")
    return cuts.astype(np.int64), cyc


def model_slab_times_case_a(stats, nnz_row, cuts, dtype: str = "float32",
                            sms: int = 148) -> np.ndarray:
    """Modeled cycles of each Case A slab [cuts[p], cuts[p+1]) (host only)."""
    lib = _lib.load()
    st = np.ascontiguousarray(stats, dtype=np.uint64)
    nz = np.ascontiguousarray(nnz_row, dtype=np.uint32)
    out = []
    for p in range(len(cuts) - 1):
        c = ctypes.c_double()
        status = lib.afmm_model_slab_time_case_a(
            _DT_CODE[dtype], nz.size, int(sms), st.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)),
            nz.ctypes.data_as(ctypes.POINTER(ctypes.c_uint32)), int(cuts[p]), int(cuts[p + 1]),
            ctypes.byref(c))
        if status != _lib.OK:
            raise InvalidArgument("afmm_model_slab_time_case_a: invalid arguments")
        out.append(c.value)
    return np.array(out)


def _gen_spec(n, density, mu_prime, integer, low, high) -> _lib.GeneratorSpec:
    spec = _lib.GeneratorSpec()
    spec.n = int(n)
    spec.density = float(density)
    spec.mu_prime = float(mu_prime)
    spec.role = _lib.ROLE_INTEGER if integer else _lib.ROLE_REAL
    spec.value_low = float(low)
    spec.value_high = float(high)
    return spec


def generate(n: int, density: float, mu_prime: float, integer: bool, seed: int,
             low: float = 0.5, high: float = 1.5, *, dtype=np.float64,
             device: Optional[int] = None) -> np.ndarray:
    """afmm::generate(GeneratorSpec, Seed) (random.hpp:111-129) on the GPU:
    the reference's matrix, bit for bit (one std::mt19937_64 stream over the
    entries in row-major order). integer=True is ValueRole::IntegerValued
    (values 1 .. 2 mu' - 1), else RealValued with bounds [low, high] (the
    reference's real_valued() sets mu' = (low + high) / 2). An invalid spec
    raises InvalidArgument with the reference's message (random.hpp:60-79)."""
    lib = _lib.load()
    dt = np.dtype(dtype)
    if dt not in (np.dtype(np.float64), np.dtype(np.float32)):
        raise InvalidArgument(f"afmm: dtype must be float32 or float64, got {dt}")
    spec = _gen_spec(n, density, mu_prime, integer, low, high)
    out = np.empty((max(int(n), 1), max(int(n), 1)), dtype=dt)
    opts, _keep = _options(ORDER_PRESERVING, device)
    err = _lib.Error()
    fn = lib.afmm_generate_f64 if dt == np.float64 else lib.afmm_generate_f32
    status = fn(ctypes.byref(spec), int(seed) & 0xFFFFFFFFFFFFFFFF, out.ctypes.data,
                ctypes.byref(opts), ctypes.byref(err))
    _raise_for(status, err)
    return out


def fp_add_peak(device: int = 0, dtype: str = "float32") -> Tuple[float, float]:
    """Measured CUDA-core FP-add peak (adds/s) and the SM clock it ran at (MHz)."""
    lib = _lib.load()
    rate = ctypes.c_double()
    mhz = ctypes.c_double()
    status = lib.afmm_fp_add_peak(int(device), _DT_CODE[dtype], ctypes.byref(rate),
                                  ctypes.byref(mhz))
    if status != _lib.OK:
        raise DeviceError("afmm_fp_add_peak failed")
    return rate.value, mhz.value


def ipc_export(tensor) -> Tuple[bytes, int]:
    """CUDA IPC handle (64 bytes) and byte offset of a device tensor's storage
    (afmm_ipc_export): another process opens it with ipc_open."""
    h = _lib.IpcHandle()
    err = _lib.Error()
    _raise_for(_lib.load().afmm_ipc_export(ctypes.c_void_p(tensor.data_ptr()), ctypes.byref(h),
                                           ctypes.byref(err)), err)
    return bytes(h.bytes), int(h.offset)


def ipc_open(device: int, handle: bytes, offset: int) -> int:
    """Map a buffer exported by another process (afmm_ipc_open); returns the
    device pointer (peer access over NVLink when the buffer is on another GPU)."""
    h = _lib.IpcHandle()
    ctypes.memmove(h.bytes, handle, 64)
    h.offset = offset
    p = ctypes.c_void_p()
    err = _lib.Error()
    _raise_for(_lib.load().afmm_ipc_open(int(device), ctypes.byref(h), ctypes.byref(p),
                                         ctypes.byref(err)), err)
    return int(p.value)


def ipc_close(ptr: int) -> None:
    _lib.load().afmm_ipc_close(ctypes.c_void_p(ptr))


def kernel_launch_count() -> int:
    return int(_lib.load().afmm_kernel_launch_count())
