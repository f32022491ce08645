"""Loading the golden vectors (tests/golden/) and regenerating their seeded inputs
with the oracle's restated generators."""
from __future__ import annotations

import hashlib
import json
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
GOLDEN_DIR = os.path.join(HERE, "golden")


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a, dtype="<f8").tobytes()).hexdigest()


def load_index() -> dict:
    with open(os.path.join(GOLDEN_DIR, "golden_index.json")) as f:
        return json.load(f)


def load_arrays() -> dict:
    with np.load(os.path.join(GOLDEN_DIR, "golden.npz")) as z:
        return {k: z[k] for k in z.files}


def regenerate(oracle, spec: dict) -> np.ndarray:
    kind = spec["kind"]
    if kind == "randint":
        return oracle.random_integer_matrix(spec["n"], spec["low"], spec["high"], spec["seed"])
    if kind == "generate":
        return oracle.generate(spec["n"], spec["density"], spec["mu"], spec["integer"],
                               spec["seed"])
    raise KeyError(kind)


def factor_pair(oracle, spec: dict):
    """bench.hpp:90-101 restated on the oracle's generator."""
    seed = spec["seed"]
    ls = oracle.splitmix64(seed)
    rs = oracle.splitmix64(seed ^ 0xD1B54A32D192ED03)
    n, d1, d2, mu = spec["n"], spec["d1"], spec["d2"], spec["mu"]
    if spec["case_b"]:
        return oracle.generate(n, d1, mu, True, ls), oracle.generate(n, d2, 1.0, False, rs)
    return oracle.generate(n, d1, 1.0, False, ls), oracle.generate(n, d2, mu, True, rs)


def seeded_inputs(oracle, entry: dict):
    specs = entry["spec"]
    if specs[0]["kind"] == "factor_pair":
        return factor_pair(oracle, specs[0])
    return regenerate(oracle, specs[0]), regenerate(oracle, specs[1])


def error_message(case: str, kind: int, row: int, col: int, value: float) -> str:
    """The reference's domain_error text (kernels.hpp:32-39) from an oracle error site."""
    where = "afmm_case_a" if case == "a" else "afmm_case_b"
    operand = "rhs" if case == "a" else "lhs"
    if kind == 1:
        return f"{where}: {operand}[{row}][{col}] = {value:f} is not integer-valued"
    return f"{where}: {operand}[{row}][{col}] exceeds the exact integer range"
