"""ctypes wrappers of the CPU checkers. TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference legs import this module; the product path (paper_1308_2400_b200/)
never does.

  Oracle     -> oracle/liboracle.so, the C restatement (afmm_oracle.c)
  FastCheck  -> oracle/libfastcheck.so, the vectorised full-size checker
                (fast_check.c; same per-element add order, pinned to the
                oracle and the reference by tests/test_oracle.py)
  Reference  -> oracle/_ref/libafmm_ref.so, the UNMODIFIED reference headers
                behind a C shim (ref_shim.cpp); built only where
                /root/reference exists, so it may be absent on a GPU box.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from ctypes import POINTER, c_char_p, c_double, c_int, c_size_t, c_uint64, c_void_p

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
FAST_SO = os.path.join(HERE, "libfastcheck.so")
REF_SO = os.path.join(HERE, "_ref", "libafmm_ref.so")


class Counts(ctypes.Structure):
    _fields_ = [("additions", c_uint64), ("multiplications", c_uint64), ("zero_skips", c_uint64)]

    def as_tuple(self):
        return (int(self.additions), int(self.multiplications), int(self.zero_skips))


class Err(ctypes.Structure):
    _fields_ = [("kind", c_int), ("row", c_uint64), ("col", c_uint64), ("value", c_double)]


def build() -> None:
    """Compile liboracle.so (and _ref when /root/reference is present)."""
    subprocess.run(["make", "-C", HERE], check=True, stdout=subprocess.DEVNULL)


class Oracle:
    """The C restatement of kernels.hpp:95-165 (+ generators)."""

    def __init__(self):
        if not os.path.exists(ORACLE_SO):
            build()
        lib = ctypes.CDLL(ORACLE_SO)
        for name in ("oracle_case_a_f64", "oracle_case_b_f64", "oracle_case_a_f32",
                     "oracle_case_b_f32"):
            f = getattr(lib, name)
            f.restype = c_int
            f.argtypes = [c_void_p, c_void_p, c_void_p, c_uint64, c_uint64, c_uint64, c_int,
                          POINTER(Counts), POINTER(Err)]
        for name in ("oracle_case_a_f64_mt", "oracle_case_b_f64_mt", "oracle_case_a_f32_mt",
                     "oracle_case_b_f32_mt"):
            f = getattr(lib, name)
            f.restype = c_int
            f.argtypes = [c_void_p, c_void_p, c_void_p, c_uint64, c_uint64, c_uint64, c_int,
                          POINTER(Counts)]
        lib.oracle_multiply_ijk_f64.argtypes = [c_void_p, c_void_p, c_void_p, c_uint64]
        lib.oracle_splitmix64.restype = c_uint64
        lib.oracle_splitmix64.argtypes = [c_uint64]
        lib.oracle_random_integer_matrix.argtypes = [c_uint64, c_int, c_int, c_uint64, c_void_p]
        lib.oracle_generate.restype = c_int
        lib.oracle_generate.argtypes = [c_uint64, c_double, c_double, c_int, c_double, c_double,
                                        c_uint64, c_void_p]
        self.lib = lib

    def product(self, case: str, lhs: np.ndarray, rhs: np.ndarray, row_begin: int = 0,
                row_end: int | None = None, validate: bool = True):
        """Returns (Z rows, (additions, multiplications, zero_skips), error-or-None)."""
        dt = lhs.dtype
        assert dt in (np.float32, np.float64) and rhs.dtype == dt
        lhs = np.ascontiguousarray(lhs)
        rhs = np.ascontiguousarray(rhs)
        n = lhs.shape[0]
        row_end = n if row_end is None else row_end
        out = np.zeros((row_end - row_begin, n), dtype=dt)
        suf = "f64" if dt == np.float64 else "f32"
        fn = getattr(self.lib, f"oracle_case_{case}_{suf}")
        c, e = Counts(), Err()
        rc = fn(lhs.ctypes.data, rhs.ctypes.data, out.ctypes.data, n, row_begin, row_end,
                1 if validate else 0, ctypes.byref(c), ctypes.byref(e))
        if rc != 0:
            return None, None, (e.kind, int(e.row), int(e.col), e.value)
        return out, c.as_tuple(), None

    def product_mt(self, case: str, lhs, rhs, row_begin: int, row_end: int, threads: int):
        dt = lhs.dtype
        n = lhs.shape[0]
        out = np.zeros((row_end - row_begin, n), dtype=dt)
        suf = "f64" if dt == np.float64 else "f32"
        fn = getattr(self.lib, f"oracle_case_{case}_{suf}_mt")
        c = Counts()
        rc = fn(lhs.ctypes.data, rhs.ctypes.data, out.ctypes.data, n, row_begin, row_end,
                int(threads), ctypes.byref(c))
        assert rc == 0
        return out, c.as_tuple()

    def multiply_ijk(self, lhs: np.ndarray, rhs: np.ndarray) -> np.ndarray:
        lhs = np.ascontiguousarray(lhs, dtype=np.float64)
        rhs = np.ascontiguousarray(rhs, dtype=np.float64)
        out = np.empty_like(lhs)
        self.lib.oracle_multiply_ijk_f64(lhs.ctypes.data, rhs.ctypes.data, out.ctypes.data,
                                         lhs.shape[0])
        return out

    def splitmix64(self, x: int) -> int:
        return int(self.lib.oracle_splitmix64(x & 0xFFFFFFFFFFFFFFFF))

    def random_integer_matrix(self, n: int, low: int, high: int, seed: int) -> np.ndarray:
        out = np.empty((n, n), dtype=np.float64)
        self.lib.oracle_random_integer_matrix(n, low, high, seed & 0xFFFFFFFFFFFFFFFF,
                                              out.ctypes.data)
        return out

    def generate(self, n: int, density: float, mu_prime: float, integer: bool, seed: int,
                 low: float = 0.5, high: float = 1.5) -> np.ndarray:
        out = np.empty((n, n), dtype=np.float64)
        rc = self.lib.oracle_generate(n, density, mu_prime, 1 if integer else 0, low, high,
                                      seed & 0xFFFFFFFFFFFFFFFF, out.ctypes.data)
        if rc != 0:
            raise ValueError("invalid GeneratorSpec")
        return out


class Reference:
    """The unmodified reference kernels via oracle/_ref/libafmm_ref.so."""

    def __init__(self):
        if not os.path.exists(REF_SO):
            raise FileNotFoundError(REF_SO)
        lib = ctypes.CDLL(REF_SO)
        for name in ("ref_afmm_case_a", "ref_afmm_case_b"):
            f = getattr(lib, name)
            f.restype = c_int
            f.argtypes = [c_void_p, c_uint64, c_void_p, c_uint64, c_void_p, POINTER(Counts),
                          c_char_p, c_size_t]
        lib.ref_multiply_ijk.restype = c_int
        lib.ref_multiply_ijk.argtypes = [c_void_p, c_void_p, c_uint64, c_void_p, POINTER(Counts),
                                         c_char_p, c_size_t]
        lib.ref_splitmix64.restype = c_uint64
        lib.ref_splitmix64.argtypes = [c_uint64]
        lib.ref_random_integer_matrix.argtypes = [c_uint64, c_int, c_int, c_uint64, c_void_p]
        lib.ref_generate.restype = c_int
        lib.ref_generate.argtypes = [c_uint64, c_double, c_double, c_int, c_double, c_double,
                                     c_uint64, c_void_p, c_char_p, c_size_t]
        lib.ref_cell_seed.restype = c_uint64
        lib.ref_cell_seed.argtypes = [c_uint64, c_uint64, c_uint64]
        lib.ref_make_factor_pair.argtypes = [c_int, c_uint64, c_double, c_double, c_double,
                                             c_uint64, c_void_p, c_void_p]
        lib.ref_make_matrix.restype = c_int
        lib.ref_make_matrix.argtypes = [c_uint64, c_char_p, c_size_t]
        lib.ref_hold_matrix.restype = c_void_p
        lib.ref_hold_matrix.argtypes = [c_void_p, c_uint64, c_char_p, c_size_t]
        lib.ref_release_matrix.argtypes = [c_void_p]
        lib.ref_run_plan_csv.restype = c_int
        lib.ref_run_plan_csv.argtypes = [c_int, c_void_p, c_size_t, c_double, c_double, c_double,
                                         c_uint64, c_uint64, c_uint64, c_char_p, c_size_t,
                                         POINTER(c_size_t), c_char_p, c_size_t]
        lib.ref_emit_table.restype = c_int
        lib.ref_emit_table.argtypes = [c_char_p, c_char_p, c_size_t, POINTER(c_size_t), c_char_p,
                                       c_size_t]
        lib.ref_case_rows.restype = c_int
        lib.ref_case_rows.argtypes = [c_int, c_void_p, c_uint64, c_uint64, c_uint64, c_void_p,
                                      c_void_p, POINTER(Counts), c_char_p, c_size_t]
        self.lib = lib

    STATUS = {0: None, 1: "shape_error", 2: "domain_error", 3: "invalid_argument", 4: "other"}

    def product(self, case: str, lhs: np.ndarray, rhs: np.ndarray):
        """Returns (Z, counts, None) or (None, None, (status_name, message))."""
        lhs = np.ascontiguousarray(lhs, dtype=np.float64)
        rhs = np.ascontiguousarray(rhs, dtype=np.float64)
        n = max(lhs.shape[0], rhs.shape[0])
        out = np.zeros((n, n), dtype=np.float64)
        c = Counts()
        msg = ctypes.create_string_buffer(512)
        fn = self.lib.ref_afmm_case_a if case == "a" else self.lib.ref_afmm_case_b
        rc = fn(lhs.ctypes.data, lhs.shape[0], rhs.ctypes.data, rhs.shape[0], out.ctypes.data,
                ctypes.byref(c), msg, 512)
        if rc != 0:
            return None, None, (self.STATUS[rc], msg.value.decode())
        return out, c.as_tuple(), None

    def run_plan_csv(self, case: str, sizes, d1: float, d2: float, mu: float, reps: int,
                     warmups: int, seed: int) -> str:
        """The reference's run_plan + emit_csv (bench.hpp:120-154, report.hpp:27-39)."""
        sz = np.ascontiguousarray(sizes, dtype=np.uint64)
        cap = 1 << 16
        while True:
            buf = ctypes.create_string_buffer(cap)
            need = c_size_t()
            msg = ctypes.create_string_buffer(512)
            rc = self.lib.ref_run_plan_csv(1 if case == "b" else 0, sz.ctypes.data, len(sz), d1,
                                           d2, mu, reps, warmups, seed, buf, cap,
                                           ctypes.byref(need), msg, 512)
            if rc == -1:
                cap = need.value
                continue
            if rc != 0:
                raise RuntimeError(msg.value.decode())
            return buf.value.decode()

    def emit_table(self, csv_text: str) -> str:
        """The reference's parse_csv + emit_table (report.hpp:74-124, 265-267)."""
        cap = 1 << 16
        while True:
            buf = ctypes.create_string_buffer(cap)
            need = c_size_t()
            msg = ctypes.create_string_buffer(512)
            rc = self.lib.ref_emit_table(csv_text.encode(), buf, cap, ctypes.byref(need), msg, 512)
            if rc == -1:
                cap = need.value
                continue
            if rc != 0:
                raise RuntimeError(msg.value.decode())
            return buf.value.decode()

    def rows_batch(self, case: str, lhs: np.ndarray, rhs: np.ndarray, blocks):
        """Run the unmodified afmm_case_{a,b} once per row block (r0, r1), all blocks
        concurrently on their own threads (ctypes releases the GIL), each on lhs with
        only its rows kept and the shared rhs. Returns (wall seconds, total additions,
        {(r0, r1): product rows})."""
        import threading
        import time

        lhs = np.ascontiguousarray(lhs, dtype=np.float64)
        rhs = np.ascontiguousarray(rhs, dtype=np.float64)
        n = lhs.shape[0]
        msg = ctypes.create_string_buffer(512)
        h = self.lib.ref_hold_matrix(rhs.ctypes.data, n, msg, 512)
        if not h:
            raise ValueError(msg.value.decode())
        out = {b: np.empty((b[1] - b[0], n), dtype=np.float64) for b in blocks}
        counts = {b: Counts() for b in blocks}
        errs = []

        def work(b):
            m = ctypes.create_string_buffer(512)
            rc = self.lib.ref_case_rows(1 if case == "b" else 0, lhs.ctypes.data, n, b[0], b[1],
                                        h, out[b].ctypes.data if b[1] > b[0] else None,
                                        ctypes.byref(counts[b]), m, 512)
            if rc != 0:
                errs.append(m.value.decode())

        threads = [threading.Thread(target=work, args=(b,)) for b in blocks]
        t0 = time.perf_counter()
        for t in threads:
            t.start()
        for t in threads:
            t.join()
        wall = time.perf_counter() - t0
        self.lib.ref_release_matrix(h)
        if errs:
            raise ValueError(errs[0])
        return wall, sum(counts[b].additions for b in blocks), out

    def multiply_ijk(self, lhs, rhs):
        lhs = np.ascontiguousarray(lhs, dtype=np.float64)
        rhs = np.ascontiguousarray(rhs, dtype=np.float64)
        out = np.empty_like(lhs)
        c = Counts()
        msg = ctypes.create_string_buffer(512)
        rc = self.lib.ref_multiply_ijk(lhs.ctypes.data, rhs.ctypes.data, lhs.shape[0],
                                       out.ctypes.data, ctypes.byref(c), msg, 512)
        assert rc == 0, msg.value
        return out

    def random_integer_matrix(self, n, low, high, seed):
        out = np.empty((n, n), dtype=np.float64)
        self.lib.ref_random_integer_matrix(n, low, high, seed & 0xFFFFFFFFFFFFFFFF,
                                           out.ctypes.data)
        return out

    def generate(self, n, density, mu_prime, integer, seed, low=0.5, high=1.5):
        out = np.empty((n, n), dtype=np.float64)
        msg = ctypes.create_string_buffer(512)
        rc = self.lib.ref_generate(n, density, mu_prime, 1 if integer else 0, low, high,
                                   seed & 0xFFFFFFFFFFFFFFFF, out.ctypes.data, msg, 512)
        if rc != 0:
            raise ValueError(msg.value.decode())
        return out

    def splitmix64(self, x):
        return int(self.lib.ref_splitmix64(x & 0xFFFFFFFFFFFFFFFF))

    def cell_seed(self, base, n, rep):
        return int(self.lib.ref_cell_seed(base, n, rep))

    def make_factor_pair(self, case_b: bool, n, d1, d2, mu, seed):
        lhs = np.empty((n, n), dtype=np.float64)
        rhs = np.empty((n, n), dtype=np.float64)
        self.lib.ref_make_factor_pair(1 if case_b else 0, n, d1, d2, mu, seed, lhs.ctypes.data,
                                      rhs.ctypes.data)
        return lhs, rhs


class FastCheck:
    """Full-size products for parity checks (fast_check.c): Case B rows
    vectorised across columns; Case A through afmm_case_a(X, Y) ==
    afmm_case_b(Y^T, X^T)^T. Inputs must be valid (the checker does not
    validate); returns Z only (counts come from the closed forms)."""

    def __init__(self):
        if not os.path.exists(FAST_SO):
            build()
        self.lib = ctypes.CDLL(FAST_SO)
        self.lib.fast_case_b_rows.restype = c_int
        self.lib.fast_case_b_rows.argtypes = [c_int, c_void_p, c_void_p, c_uint64, c_void_p,
                                              c_uint64, c_void_p, c_int]

    def case_b_rows(self, lhs: np.ndarray, rhs: np.ndarray, rows, threads: int = 0) -> np.ndarray:
        """Rows `rows` (any row indices, or a (r0, r1) range) of afmm_case_b(lhs, rhs)."""
        dt = lhs.dtype
        assert rhs.dtype == dt and dt in (np.float32, np.float64)
        lhs = np.ascontiguousarray(lhs)
        rhs = np.ascontiguousarray(rhs)
        n = lhs.shape[0]
        if isinstance(rows, tuple):
            rows = np.arange(rows[0], rows[1])
        idx = np.ascontiguousarray(rows, dtype=np.uint64)
        z = np.empty((idx.size, n), dtype=dt)
        rc = self.lib.fast_case_b_rows(0 if dt == np.float64 else 1, lhs.ctypes.data,
                                       rhs.ctypes.data, n, idx.ctypes.data, idx.size,
                                       z.ctypes.data, threads or os.cpu_count() or 1)
        if rc != 0:
            raise RuntimeError("fast_case_b_rows failed")
        return z

    def product(self, case: str, lhs: np.ndarray, rhs: np.ndarray, threads: int = 0) -> np.ndarray:
        """The whole n x n product."""
        n = lhs.shape[0]
        if case == "b":
            return self.case_b_rows(lhs, rhs, (0, n), threads)
        zt = self.case_b_rows(np.ascontiguousarray(rhs.T), np.ascontiguousarray(lhs.T), (0, n),
                              threads)
        return np.ascontiguousarray(zt.T)


def reference_available() -> bool:
    return os.path.exists(REF_SO)


def ref_b16_pair(ref: Reference):
    """test_kernels.cpp:208-217 operands, from the reference's own RNG calls."""
    lhs = np.empty((8, 8), dtype=np.float64)
    rhs = np.empty((8, 8), dtype=np.float64)
    ref.lib.ref_b16_pair.argtypes = [c_void_p, c_void_p]
    ref.lib.ref_b16_pair(lhs.ctypes.data, rhs.ctypes.data)
    return lhs, rhs
