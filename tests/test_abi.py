"""The C-ABI library without a GPU: it loads, exports every symbol include/afmm_b200.h
declares, and its host-side logic (dimension checks, row partition) behaves as the
reference's contract says. No compute call is made here."""
import ctypes
import os
import re
import shutil
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "afmm_b200.h")


def _declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:[\w\s\*]+?)\b(afmm_\w+)\s*\(", text, re.M)))


def test_library_exports_every_declared_symbol():
    from paper_1308_2400_b200 import _lib

    lib = _lib.load()
    declared = _declared_symbols()
    assert len(declared) >= 15
    for name in declared:
        assert hasattr(lib, name), name
    assert set(declared) == set(_lib.EXPORTED_SYMBOLS)
    assert lib.afmm_abi_version() == _lib.ABI_VERSION == 2


def test_library_is_sm100a_only():
    """The product .so carries sm_100a SASS (no PTX JIT, no other arch)."""
    cuobjdump = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(cuobjdump):
        pytest.skip("cuobjdump not available")
    from paper_1308_2400_b200 import _lib

    out = subprocess.run([cuobjdump, "--list-elf", _lib.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run([cuobjdump, "-sass", _lib.LIB_PATH], capture_output=True,
                          text=True).stdout
    for mnemonic in ("UTMALDG", "FADD2", "DADD", "SYNCS.PHASECHK"):
        assert mnemonic in sass, mnemonic
    assert "HMMA" not in sass and "UTCHMMA" not in sass  # no tensor cores: no multiplications


def test_status_strings():
    from paper_1308_2400_b200 import _lib

    assert _lib.status_string(_lib.OK) == "ok"
    assert _lib.status_string(_lib.ERR_SHAPE) == "shape_error"
    assert _lib.status_string(_lib.ERR_DOMAIN) == "domain_error"


def test_dimension_mismatch_is_shape_error_before_any_device_work():
    import paper_1308_2400_b200 as afmm

    with pytest.raises(afmm.ShapeError) as ei:
        afmm.afmm_case_a(np.zeros((2, 2)), np.zeros((3, 3)))
    assert str(ei.value) == "afmm_case_a: dimension mismatch 2 vs 3"
    with pytest.raises(afmm.ShapeError) as ei:
        afmm.afmm_case_b(np.zeros((2, 2)), np.zeros((3, 3)))
    assert str(ei.value) == "afmm_case_b: dimension mismatch 2 vs 3"
    assert issubclass(afmm.ShapeError, ValueError)  # shape_error : std::invalid_argument


def test_empty_matrix_is_invalid_argument():
    import paper_1308_2400_b200 as afmm

    with pytest.raises(afmm.InvalidArgument) as ei:
        afmm.afmm_case_b(np.zeros((0, 0)), np.zeros((0, 0)))
    assert str(ei.value) == "DenseMatrix: dimension must be >= 1"


def test_mode_codes_and_unknown_mode_rejected():
    """The three modes of afmm_options.mode (include/afmm_b200.h) and an unknown
    code: rejected by the C ABI before any device work."""
    import ctypes

    import paper_1308_2400_b200 as afmm
    from paper_1308_2400_b200 import _lib

    assert (_lib.MODE_ORDER_PRESERVING, _lib.MODE_FAST, _lib.MODE_FAST_LADDER) == (0, 1, 2)
    assert afmm.FAST_LADDER == "fast-ladder"
    with pytest.raises(afmm.InvalidArgument):
        afmm.afmm_case_a(np.eye(2), np.eye(2), mode="reassociate-everything")
    lib = _lib.load()
    o = _lib.Options()
    o.mode = 3
    o.device = -1
    x = np.eye(2)
    z = np.empty_like(x)
    c, e = _lib.OpCounts(), _lib.Error()
    st = lib.afmm_case_a_f64(x.ctypes.data, 2, x.ctypes.data, 2, z.ctypes.data, ctypes.byref(o),
                             ctypes.byref(c), ctypes.byref(e))
    assert st == _lib.ERR_INVALID_ARGUMENT
    assert b"options.mode" in bytes(e.message)


def test_ladder_additions_closed_form():
    """gen.ladder_additions (the adds the fast-ladder mode performs) against a
    direct count: floor(log2 r) + popcount(r) per nonzero rep and nonzero base."""
    from paper_1308_2400_b200.gen import expected_additions, ladder_additions

    rng = np.random.default_rng(2)
    n = 23
    reps = rng.integers(-40, 41, size=(n, n)).astype(np.float64)
    bases = rng.standard_normal((n, n)) * (rng.random((n, n)) < 0.6)
    cost = lambda r: 0 if r == 0 else (abs(r).bit_length() - 1) + bin(abs(r)).count("1")
    want_b = sum(cost(int(reps[i, k])) * int((bases[k] != 0).sum())
                 for i in range(n) for k in range(n))
    assert ladder_additions("b", reps, bases) == want_b
    want_a = sum(cost(int(reps[k, j])) for i in range(n) for k in range(n) if bases[i, k] != 0
                 for j in range(n))
    assert ladder_additions("a", bases, reps) == want_a
    assert ladder_additions("b", reps, bases) < expected_additions("b", reps, bases)


def test_no_cpu_fallback_without_a_device():
    """Without a CUDA device the product must fail loudly, never compute on the host."""
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    import paper_1308_2400_b200 as afmm

    with pytest.raises(afmm.DeviceError):
        afmm.afmm_case_a(np.eye(2), np.eye(2))


@pytest.mark.parametrize("parts", [1, 2, 3, 4, 8])
def test_partition_rows_balanced_and_monotone(parts):
    from paper_1308_2400_b200 import partition_rows

    rng = np.random.default_rng(parts)
    for n in (1, 5, 64, 1000):
        w = rng.integers(0, 10_000, n).astype(np.uint64)
        w[rng.random(n) < 0.2] = 0
        cuts = partition_rows(w, parts)
        assert cuts[0] == 0 and cuts[-1] == n and len(cuts) == parts + 1
        assert np.all(np.diff(cuts) >= 0)
        total = int(w.sum())
        for p in range(parts):
            s = int(w[cuts[p]:cuts[p + 1]].sum())
            # each part is within one row's work of its fair share
            assert abs(s - total / parts) <= int(w.max()) + 1, (n, parts, p)


def test_partition_rows_skewed_beta_rows():
    """cfg4-like skew: Beta(0.5,0.5) row densities; cuts follow work, not row count."""
    from paper_1308_2400_b200 import partition_rows

    rng = np.random.default_rng(0)
    w = (rng.beta(0.5, 0.5, 8192) * 1e6).astype(np.uint64)
    cuts = partition_rows(w, 8)
    shares = [int(w[cuts[p]:cuts[p + 1]].sum()) for p in range(8)]
    assert max(shares) / min(shares) < 1.005  # one row of work is ~0.2% of a share


def test_cpp_wrapper_header_compiles():
    """include/afmm_b200/kernels.hpp against the reference's own headers (drop-in check)."""
    ref_inc = "/root/reference/proj/include"
    if not os.path.isdir(ref_inc):
        pytest.skip("reference headers not present")
    src = (
        '#include "afmm_b200/kernels.hpp"\n'
        "int main() {\n"
        "  afmm::DenseMatrix x(2), y(2);\n"
        "  auto (*fa)(const afmm::DenseMatrix&, const afmm::DenseMatrix&, afmm::gpu::Options)"
        " -> afmm::MultiplyResult = &afmm::gpu::afmm_case_a;\n"
        "  (void)fa; (void)x; (void)y;\n"
        "  return afmm::gpu::parse_kernel(\"afmm-a-gpu\").has_value() ? 0 : 1;\n}\n")
    r = subprocess.run(["g++", "-std=c++20", "-fsyntax-only", "-x", "c++", "-I", ref_inc, "-I",
                        os.path.join(ROOT, "include"), "-"], input=src, capture_output=True,
                       text=True)
    assert r.returncode == 0, r.stderr


def test_bench_refuses_more_gpus_than_visible():
    """`bench.py --gpus N` without torchrun drives N devices in one process; it
    refuses (exit 2, no JSON line) when fewer are visible instead of timing one
    GPU under an N-GPU label."""
    import sys

    import torch

    if torch.cuda.device_count() >= 4:
        pytest.skip("enough GPUs")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "4",
                        "--steps", "1", "--warmup", "3", "--size", "64"], cwd=ROOT,
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 2
    assert not [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert "refusing" in r.stderr


def test_case_a_cut_by_modeled_time_balances_sorted_density_rows():
    """cfg4's Case A (per-row densities from Beta(0.5, 0.5)) with the rows
    SORTED by density. The cut by modeled time (the device-side A-form /
    B-form choice evaluated per slab, tile and wave quantisation included)
    balances what an equal-row cut leaves lopsided: at 8 devices the slabs'
    modeled times are within 7% of each other (equal rows: the sparsest slab
    takes 1/9 of the densest one's time) and at 2 devices the makespan drops.
    The residual: each dense slab costs one whole B-form tile (1024 rows)
    whatever its row count, and the sparse slab's A-form time jumps by a wave
    exactly where it would catch up. Host-only model query."""
    import paper_1308_2400_b200 as afmm
    from paper_1308_2400_b200.gen import make_inputs

    lhs, rhs = make_inputs("cfg4", seed=0, n=8192)
    order = np.argsort((lhs != 0).sum(axis=1), kind="stable")
    lhs = np.ascontiguousarray(lhs[order])
    stats, nnz_row = afmm.case_a_statistics(lhs, rhs)
    for parts in (8, 2):
        cuts, cyc = afmm.model_partition_case_a(stats, nnz_row, parts)
        assert cuts[0] == 0 and cuts[-1] == 8192 and np.all(np.diff(cuts) > 0)
        assert np.allclose(cyc, afmm.model_slab_times_case_a(stats, nnz_row, cuts))
        equal = np.linspace(0, 8192, parts + 1).astype(np.int64)
        t_equal = afmm.model_slab_times_case_a(stats, nnz_row, equal)
        assert cyc.max() <= t_equal.max() * 1.0001
        if parts == 8:
            assert cyc.max() / cyc.min() <= 1.07, (cuts, cyc)
            assert t_equal.max() / t_equal.min() > 5
        else:
            assert cyc.max() < t_equal.max() * 0.99, (cyc, t_equal)


def test_case_a_statistics_match_the_closed_forms():
    import paper_1308_2400_b200 as afmm

    rng = np.random.default_rng(3)
    x = rng.standard_normal((70, 70)) * (rng.random((70, 70)) < 0.3)
    y = rng.integers(-3000, 3000, (70, 70)).astype(np.float64)
    y[0, 0] = 2.5  # llround(2.5) = 3 (half away from zero)
    stats, nnz = afmm.case_a_statistics(x, y)
    r = np.where(np.abs(y - np.trunc(y)) == 0.5, np.trunc(y) + np.sign(y), np.rint(y))
    assert int(stats[0]) == int((r != 0).sum())
    assert int(stats[2]) == int((np.abs(r) > 2048).sum())
    assert int(stats[3]) == int(np.abs(r).sum())
    assert int(stats[1]) == int(np.minimum(np.abs(r), 2048).max(axis=1).sum())
    assert np.array_equal(nnz, (x != 0).sum(axis=1))
