"""Generate the golden vectors in tests/golden/ from the UNMODIFIED reference.

Run in the build container (where /root/reference exists):

    make -C oracle && python tests/golden/make_golden.py

Every expected product, OpCounts and error message below comes from the
reference's own afmm_case_a / afmm_case_b (kernels.hpp:113-165), called through
oracle/_ref/libafmm_ref.so (oracle/ref_shim.cpp over the reference headers as
they lie in /root/reference/proj/include). Inputs come from the reference's own
generators (random.hpp:111-129, test_kernels.cpp:16-24, acceptance.hpp:72-82,
bench.hpp:82-101) or, for edge cases the reference tests do not generate,
from numpy with a fixed seed; those inputs are stored verbatim.

Outputs:
  golden.npz          arrays of the stored fixtures ("<name>/lhs|rhs|z")
  golden_index.json   per fixture: case, counts or error; per seeded case:
                      generator spec + sha256 of lhs, rhs and product bytes
"""
from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle.oracle import Reference, ref_b16_pair  # noqa: E402

M64 = 0xFFFFFFFFFFFFFFFF


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a, dtype="<f8").tobytes()).hexdigest()


def main() -> None:
    ref = Reference()
    arrays: dict[str, np.ndarray] = {}
    fixtures = []
    seeded = []

    def stored(name, case, lhs, rhs, source):
        lhs = np.asarray(lhs, dtype=np.float64)
        rhs = np.asarray(rhs, dtype=np.float64)
        z, counts, err = ref.product(case, lhs, rhs)
        arrays[f"{name}/lhs"] = lhs
        arrays[f"{name}/rhs"] = rhs
        entry = {"name": name, "case": case, "source": source}
        if err is None:
            arrays[f"{name}/z"] = z
            entry["counts"] = list(counts)
        else:
            entry["error"] = {"type": err[0], "message": err[1]}
        fixtures.append(entry)

    # --- test_kernels.cpp hand traces, degenerate and error cases -----------------
    stored("a_hand_trace", "a", [[2, 0], [0.5, 1]], [[3, 1], [0, 2]], "test_kernels.cpp:109-115")
    stored("a_all_zero", "a", np.zeros((3, 3)), [[1, 2, 3], [4, 5, 6], [7, 8, 9]],
           "test_kernels.cpp:117-121")
    stored("a_identity", "a", np.eye(3), [[1, -2, 0], [3, 0, 4], [0, 5, -6]],
           "test_kernels.cpp:123-126")
    stored("a_dim_mismatch", "a", np.zeros((2, 2)), np.zeros((3, 3)), "test_kernels.cpp:130")
    stored("a_not_integer", "a", np.zeros((2, 2)), [[1, 0.5], [0, 2]], "test_kernels.cpp:131-132")
    stored("a_near_integer", "a", np.eye(2), [[1 + 1e-12, 0], [0, 2 - 1e-12]],
           "test_kernels.cpp:134-135")
    stored("b_hand_trace", "b", [[3, 0], [1, 2]], [[0.5, 0], [1, 1]], "test_kernels.cpp:175-186")
    stored("b_all_zero", "b", np.zeros((3, 3)), [[1, 2, 3], [4, 5, 6], [7, 8, 9]],
           "test_kernels.cpp:189-191")
    stored("b_dim_mismatch", "b", np.zeros((2, 2)), np.zeros((3, 3)), "test_kernels.cpp:193")
    stored("b_not_integer", "b", [[1, 0], [0.25, 2]], np.zeros((2, 2)), "test_kernels.cpp:194-195")
    b16_l, b16_r = ref_b16_pair(ref)
    stored("a_b16", "a", b16_l, b16_r, "test_kernels.cpp:208-223")
    stored("b_b16", "b", b16_l, b16_r, "test_kernels.cpp:208-223")

    # --- reps beyond int32 (accepted by the reference up to 2^53, kernels.hpp:36-39);
    # the device splits them into consecutive list entries at the same k --------------
    huge = float(2 ** 31 + 5)
    stored("a_rep_2p31_plus_5", "a", [[0.5, -0.25], [1e-3, 3.0]], [[1, huge], [-2, 0]],
           "kernels.hpp:36-39, 95-104 (|rep| > 2^31 - 1)")
    stored("b_rep_2p31_plus_5", "b", [[1, -2], [huge, 0]], [[0.5, -0.25], [1e-3, 3.0]],
           "kernels.hpp:36-39, 95-104 (|rep| > 2^31 - 1)")
    stored("a_rep_2p31_plus_5_n1", "a", [[-0.375]], [[huge]],
           "kernels.hpp:36-39 (one list needs 2 entries > n: capacity re-run)")

    # --- range / sign / zero edge cases (kernels.hpp:25-43, :95-104) -------------
    big = 2.0 ** 53 + 2.0
    stored("a_out_of_range", "a", np.eye(2), [[1, 0], [big, 2]], "kernels.hpp:36-39")
    stored("b_out_of_range", "b", [[1, 0], [0, -big]], np.eye(2), "kernels.hpp:36-39")
    stored("a_first_offender_order", "a", np.eye(3), [[1, 2, 3], [4, 5.5, 6], [7.25, 8, 9]],
           "kernels.hpp:27-29 (row-major first offender)")
    stored("b_kind_at_first", "b", [[1, 2, 3], [4, big, 6], [7.5, 8, 9]], np.eye(3),
           "kernels.hpp:31-39 (range error before a later non-integer)")
    stored("a_negative_reps", "a", [[1.5, -2.25], [0.125, 3]], [[-3, 2], [1, -4]],
           "kernels.hpp:97-99")
    stored("b_negative_reps", "b", [[-3, 2], [1, -4]], [[1.5, -2.25], [0.125, 3]],
           "kernels.hpp:97-99")
    stored("a_neg_zero_base", "a", [[-0.0, 1.0], [2.0, -0.0]], [[5, -3], [-7, 1]],
           "kernels.hpp:122 (-0.0 == 0.0 is a zero base)")
    stored("b_neg_zero_base", "b", [[5, -3], [-7, 1]], [[-0.0, 1.0], [2.0, -0.0]],
           "kernels.hpp:156")
    stored("a_tiny_rep_rounds_to_zero", "a", [[1.0, 2.0], [3.0, 4.0]], [[1e-12, 2], [-1e-12, 0]],
           "kernels.hpp:129-130 (llround == 0 skipped, not tallied)")
    stored("b_tiny_rep_rounds_to_zero", "b", [[1e-12, 2], [-1e-12, 0]], [[1.0, 2.0], [3.0, 4.0]],
           "kernels.hpp:152-153")
    stored("a_n1", "a", [[0.75]], [[7]], "n = 1")
    stored("b_n1", "b", [[-7]], [[0.75]], "n = 1")
    stored("a_n1_zero", "a", [[0.0]], [[7]], "n = 1 zero base")

    # --- survey identity-probe style randomized cases (stored inputs) -------------
    rng = np.random.default_rng(1308_2400)
    for n in (1, 2, 3, 5, 8, 17, 33, 64):
        for rep_i in range(2):
            u = rng.random((n, n))
            bases = rng.uniform(-4, 4, (n, n))
            bases[u < 0.30] = 0.0
            bases[(u >= 0.30) & (u < 0.35)] = -0.0
            bases[(u >= 0.35) & (u < 0.40)] = 1e-300
            v = rng.random((n, n))
            reps = rng.integers(-20, 21, (n, n)).astype(np.float64)
            reps[v < 0.30] = 0.0
            reps[(v >= 0.30) & (v < 0.33)] = 1e-12
            stored(f"a_probe_n{n}_{rep_i}", "a", bases, reps, "SURVEY.md appendix probe 3")
            stored(f"b_probe_n{n}_{rep_i}", "b", reps, bases, "SURVEY.md appendix probe 3")

    # --- seeded cases regenerated from the restated generators --------------------
    def seeded_case(name, case, lhs, rhs, spec):
        z, counts, err = ref.product(case, lhs, rhs)
        assert err is None, err
        seeded.append({"name": name, "case": case, "spec": spec, "lhs_sha": sha(lhs),
                       "rhs_sha": sha(rhs), "z_sha": sha(z), "counts": list(counts)})

    # test_kernels.cpp:138-147 (Case A integer) and :198-206 (Case B integer)
    for seed in range(10):
        spec_l = {"kind": "randint", "n": 16, "low": -9, "high": 9, "seed": seed * 2 + 1}
        spec_r = {"kind": "randint", "n": 16, "low": -9, "high": 9, "seed": seed * 2 + 2}
        seeded_case(f"tk_a_int_{seed}", "a", ref.random_integer_matrix(16, -9, 9, seed * 2 + 1),
                    ref.random_integer_matrix(16, -9, 9, seed * 2 + 2), [spec_l, spec_r])
        spec_l = {"kind": "randint", "n": 16, "low": -9, "high": 9, "seed": seed * 3 + 1}
        spec_r = {"kind": "randint", "n": 16, "low": -9, "high": 9, "seed": seed * 3 + 2}
        seeded_case(f"tk_b_int_{seed}", "b", ref.random_integer_matrix(16, -9, 9, seed * 3 + 1),
                    ref.random_integer_matrix(16, -9, 9, seed * 3 + 2), [spec_l, spec_r])
    # test_kernels.cpp:149-155 (real x integer, Case A)
    for seed in range(10):
        sl = {"kind": "generate", "n": 32, "density": 0.9, "mu": 1.0, "integer": False,
              "seed": seed}
        sr = {"kind": "generate", "n": 32, "density": 0.8, "mu": 21.0, "integer": True,
              "seed": seed + 31}
        seeded_case(f"tk_a_real_{seed}", "a", ref.generate(32, 0.9, 1.0, False, seed),
                    ref.generate(32, 0.8, 21.0, True, seed + 31), [sl, sr])
    # acceptance.hpp:93-118 (c01: 350 integer pairs, both cases)
    for n in (1, 2, 3, 8, 16, 33, 64):
        for pair in range(50):
            key = ref.splitmix64((n << 32) | pair)
            s1, s2 = ref.splitmix64(key), ref.splitmix64(key ^ 1)
            lhs = ref.random_integer_matrix(n, -9, 9, s1)
            rhs = ref.random_integer_matrix(n, -9, 9, s2)
            spec = [{"kind": "randint", "n": n, "low": -9, "high": 9, "seed": s1},
                    {"kind": "randint", "n": n, "low": -9, "high": 9, "seed": s2}]
            seeded_case(f"c01_a_n{n}_{pair}", "a", lhs, rhs, spec)
            seeded_case(f"c01_b_n{n}_{pair}", "b", lhs, rhs, spec)
    # acceptance.hpp:121-139 (c02: 50 real x integer pairs, Case A)
    for s in range(50):
        n = (8, 16, 33, 64)[s % 4]
        mu = (1, 3, 5, 7, 14, 21)[s % 6]
        ls, rs = ref.splitmix64(0xA11CE + s), ref.splitmix64(0xB0B + s)
        sl = {"kind": "generate", "n": n, "density": 0.7, "mu": 1.0, "integer": False, "seed": ls}
        sr = {"kind": "generate", "n": n, "density": 0.5, "mu": float(mu), "integer": True,
              "seed": rs}
        seeded_case(f"c02_a_{s}", "a", ref.generate(n, 0.7, 1.0, False, ls),
                    ref.generate(n, 0.5, float(mu), True, rs), [sl, sr])
    # acceptance.hpp:170-190 (c04 inputs, both cases)
    for n in (5, 17, 32):
        for s in range(10):
            a1, a2 = ref.splitmix64(0xC4F + n + s), ref.splitmix64(0xD4F + n + s)
            il, ir = ref.random_integer_matrix(n, -9, 9, a1), ref.random_integer_matrix(n, -9, 9, a2)
            spec = [{"kind": "randint", "n": n, "low": -9, "high": 9, "seed": a1},
                    {"kind": "randint", "n": n, "low": -9, "high": 9, "seed": a2}]
            seeded_case(f"c04_a_int_n{n}_{s}", "a", il, ir, spec)
            seeded_case(f"c04_b_int_n{n}_{s}", "b", il, ir, spec)
            r1, r2 = ref.splitmix64(0xE4F + n + s), ref.splitmix64(0xF4F + n + s)
            rl = ref.generate(n, 0.6, 1.0, False, r1)
            ic = ref.generate(n, 0.4, 3.0, True, r2)
            sl = {"kind": "generate", "n": n, "density": 0.6, "mu": 1.0, "integer": False,
                  "seed": r1}
            sr = {"kind": "generate", "n": n, "density": 0.4, "mu": 3.0, "integer": True,
                  "seed": r2}
            seeded_case(f"c04_a_real_n{n}_{s}", "a", rl, ic, [sl, sr])
            seeded_case(f"c04_b_real_n{n}_{s}", "b", ic, rl, [sr, sl])
    # bench.hpp:82-101 factor pairs (the reference's bench/c03 inputs)
    for case, n, d1, d2, mu in (("a", 64, 1 / 3, 0.5, 3.0), ("a", 64, 0.2, 0.4, 14.0),
                                ("b", 48, 0.5, 0.7, 7.0)):
        for rep in range(3):
            cs = ref.cell_seed(7001, n, rep)
            lhs, rhs = ref.make_factor_pair(case == "b", n, d1, d2, mu, cs)
            seeded_case(f"pair_{case}_n{n}_mu{int(mu)}_{rep}", case, lhs, rhs,
                        [{"kind": "factor_pair", "case_b": case == "b", "n": n, "d1": d1,
                          "d2": d2, "mu": mu, "seed": cs}])

    np.savez_compressed(os.path.join(HERE, "golden.npz"), **arrays)
    with open(os.path.join(HERE, "golden_index.json"), "w") as f:
        json.dump({"generator": "tests/golden/make_golden.py",
                   "reference": "/root/reference/proj/include/afmm (unmodified)",
                   "fixtures": fixtures, "seeded": seeded}, f, indent=1)
    print(f"{len(fixtures)} stored fixtures, {len(seeded)} seeded cases")


if __name__ == "__main__":
    main()
