"""Pins the CPU oracle (oracle/afmm_oracle.c) to the reference before it is trusted.

(1) golden vectors produced by the unmodified reference (tests/golden/),
(2) the live reference library oracle/_ref when it is built (this container),
(3) the algebraic facts the GPU design relies on (transposition identity,
    closed-form counts), checked on the oracle itself.
"""
import numpy as np
import pytest

from golden_util import error_message, load_arrays, load_index, seeded_inputs, sha

INDEX = load_index()
ARRAYS = load_arrays()


@pytest.mark.parametrize("fx", INDEX["fixtures"], ids=[f["name"] for f in INDEX["fixtures"]])
def test_oracle_matches_golden_fixture(oracle, fx):
    lhs = ARRAYS[fx["name"] + "/lhs"]
    rhs = ARRAYS[fx["name"] + "/rhs"]
    if "error" in fx and fx["error"]["type"] == "shape_error":
        assert lhs.shape != rhs.shape  # the oracle takes one n; shape errors are host logic
        return
    z, counts, err = oracle.product(fx["case"], lhs, rhs)
    if "error" in fx:
        assert err is not None
        assert error_message(fx["case"], *err) == fx["error"]["message"]
        return
    assert err is None
    assert counts == tuple(fx["counts"])
    exp = ARRAYS[fx["name"] + "/z"]
    assert np.array_equal(z.view(np.uint64), exp.view(np.uint64)), "not bit-identical"


def test_oracle_matches_golden_seeded(oracle):
    """909 seeded cases: c01 (350 pairs x 2 cases), c02, c04, test_kernels loops, bench pairs."""
    for entry in INDEX["seeded"]:
        lhs, rhs = seeded_inputs(oracle, entry)
        assert sha(lhs) == entry["lhs_sha"], entry["name"]
        assert sha(rhs) == entry["rhs_sha"], entry["name"]
        z, counts, err = oracle.product(entry["case"], lhs, rhs)
        assert err is None
        assert counts == tuple(entry["counts"]), entry["name"]
        assert sha(z) == entry["z_sha"], entry["name"]


def _random_case(rng, n):
    u = rng.random((n, n))
    bases = rng.uniform(-4, 4, (n, n))
    bases[u < 0.3] = 0.0
    bases[(u >= 0.3) & (u < 0.35)] = -0.0
    v = rng.random((n, n))
    reps = rng.integers(-12, 13, (n, n)).astype(np.float64)
    reps[v < 0.25] = 0.0
    reps[(v >= 0.25) & (v < 0.28)] = -1e-12
    return bases, reps


def test_oracle_matches_live_reference(oracle, reference):
    rng = np.random.default_rng(77)
    for n in (1, 4, 9, 31, 50):
        for _ in range(3):
            bases, reps = _random_case(rng, n)
            for case, lhs, rhs in (("a", bases, reps), ("b", reps, bases)):
                zr, cr, er = reference.product(case, lhs, rhs)
                zo, co, eo = oracle.product(case, lhs, rhs)
                assert er is None and eo is None
                assert co == cr
                assert np.array_equal(zo.view(np.uint64), zr.view(np.uint64))


def test_oracle_generators_match_reference(oracle, reference):
    for seed in (0, 1, 12345, 2**63 + 5):
        assert oracle.splitmix64(seed) == reference.splitmix64(seed)
        assert np.array_equal(oracle.random_integer_matrix(9, -9, 9, seed),
                              reference.random_integer_matrix(9, -9, 9, seed))
        assert np.array_equal(oracle.generate(11, 0.4, 7.0, True, seed),
                              reference.generate(11, 0.4, 7.0, True, seed))
        assert np.array_equal(oracle.generate(11, 0.8, 1.0, False, seed, -1.0, 2.0),
                              reference.generate(11, 0.8, 1.0, False, seed, -1.0, 2.0))


def test_f32_restatement_exact_on_representable_inputs(oracle, reference):
    """The reference is fp64-only (proj/README.md:91). On inputs whose every partial
    sum is exact in fp32 (small integers x dyadic bases) the fp32 restatement must
    equal the unmodified fp64 reference bit-for-bit once widened."""
    rng = np.random.default_rng(5)
    for n in (3, 16, 40):
        bases = rng.integers(-64, 65, (n, n)) / 8.0
        bases[rng.random((n, n)) < 0.3] = 0.0
        reps = rng.integers(-9, 10, (n, n)).astype(np.float64)
        for case, lhs, rhs in (("a", bases, reps), ("b", reps, bases)):
            zr, cr, _ = reference.product(case, lhs, rhs)
            zo, co, _ = oracle.product(case, lhs.astype(np.float32), rhs.astype(np.float32))
            assert co == cr
            assert np.array_equal(zo.astype(np.float64), zr)


def test_transposition_identity(oracle):
    """afmm_case_a(X, Y) == afmm_case_b(Y^T, X^T)^T bit-for-bit with identical additions:
    the per-element add sequence (k ascending, |rep| copies) is the same. This is
    what lets the GPU run Case A through the warp-uniform Case-B kernel."""
    rng = np.random.default_rng(11)
    for n in (1, 2, 5, 17, 33):
        for _ in range(4):
            bases, reps = _random_case(rng, n)
            for dt in (np.float64, np.float32):
                x, y = bases.astype(dt), reps.astype(dt)
                za, ca, _ = oracle.product("a", x, y)
                zb, cb, _ = oracle.product("b", np.ascontiguousarray(y.T), np.ascontiguousarray(x.T))
                assert np.array_equal(za.view(np.uint8), np.ascontiguousarray(zb.T).view(np.uint8))
                assert ca[0] == cb[0]


def test_closed_form_counts(oracle):
    """SURVEY.md 8.0 closed forms, which the device prepass computes."""
    rng = np.random.default_rng(3)
    for n in (1, 3, 8, 21):
        for _ in range(5):
            bases, reps = _random_case(rng, n)
            r = np.abs(np.array([[round(v) if abs(v) >= 0.5 else 0 for v in row] for row in reps]))
            # Case A: additions = sum_{(i,k): X != 0} sum_j |llround Y[k,j]|
            _, ca, _ = oracle.product("a", bases, reps)
            nzx = bases != 0
            assert ca[0] == int((nzx.sum(axis=0) * r.sum(axis=1)).sum())
            assert ca[2] == int((~nzx).sum())
            # Case B: additions = sum |llround X[i,k]| * nnz(Y[k,:])
            _, cb, _ = oracle.product("b", reps, bases)
            nnzb = (bases != 0).sum(axis=1)
            assert cb[0] == int((r.sum(axis=0) * nnzb).sum())
            assert cb[2] == int(((r != 0) * (n - nnzb)[None, :]).sum())


def test_row_slab_and_threads_are_bit_identical(oracle):
    rng = np.random.default_rng(9)
    bases, reps = _random_case(rng, 37)
    for case, lhs, rhs in (("a", bases, reps), ("b", reps, bases)):
        z, c, _ = oracle.product(case, lhs, rhs)
        zs, cs, _ = oracle.product(case, lhs, rhs, 5, 23)
        assert np.array_equal(zs, z[5:23])
        zm, cm = oracle.product_mt(case, lhs, rhs, 0, 37, 4)
        assert np.array_equal(zm.view(np.uint64), z.view(np.uint64)) and cm == c


@pytest.mark.parametrize("seed", range(4))
def test_fast_checker_is_bit_identical_to_the_oracle(oracle, seed):
    """oracle/fast_check.c (the vectorised full-size checker) against the
    scalar restatement: both cases, fp32/fp64, ragged n (chunk tails), signed
    reps, zero / -0.0 / subnormal bases, overflow to +/-inf, any row list."""
    from oracle.oracle import FastCheck

    fc = FastCheck()
    rng = np.random.default_rng(600 + seed)
    for n in (1, 3, 31, 65, 257, 300):
        for dt in (np.float32, np.float64):
            bases = rng.standard_normal((n, n)) * (rng.random((n, n)) < 0.6)
            u = rng.random((n, n))
            bases[u < 0.05] = -0.0
            bases[(u > 0.05) & (u < 0.08)] = np.finfo(dt).tiny / 7
            if seed == 3:
                bases *= np.finfo(dt).max / 8
            reps = rng.integers(-9, 10, (n, n)) * (rng.random((n, n)) < 0.7)
            bases, reps = bases.astype(dt), reps.astype(dt)
            for case, lhs, rhs in (("a", bases, reps), ("b", reps, bases)):
                z, c, _ = oracle.product(case, lhs, rhs)
                zf = fc.product(case, lhs, rhs, threads=3)
                assert np.array_equal(z.view(np.uint8), zf.view(np.uint8)), (n, dt, case)
                if case == "b":
                    rows = rng.integers(0, n, min(n, 37))
                    zr = fc.case_b_rows(lhs, rhs, rows, threads=2)
                    assert np.array_equal(zr.view(np.uint8), z[rows].view(np.uint8))


def test_fast_checker_matches_live_reference(reference):
    """The checker against the unmodified reference (fp64) on a BASELINE-like
    Case B and Case A input."""
    from oracle.oracle import FastCheck
    from paper_1308_2400_b200.gen import expected_counts, make_inputs

    fc = FastCheck()
    for name, case in (("cfg2", "b"), ("cfg1", "a")):
        lhs, rhs = make_inputs(name, seed=5, n=160)
        z, c, err = reference.product(case, lhs, rhs)
        assert err is None
        assert np.array_equal(z.view(np.uint8), fc.product(case, lhs, rhs).view(np.uint8))
        assert c == expected_counts(case, lhs, rhs)
