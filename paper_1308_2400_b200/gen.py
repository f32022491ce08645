"""Seeded synthetic inputs for the BASELINE.json configurations.

There is no dataset behind this path: BASELINE.json's configs describe value
distributions, and these generators reproduce them with a seeded numpy PCG64
stream (not the reference's mt19937_64 bit maps, random.hpp:92-104, which
cannot express N(0,1), Beta or geometric draws). The same host buffers feed
the GPU product and the CPU oracle, so parity never depends on the generator.

Pinned interpretations of ambiguous wording (DESIGN.md repeats them):
  * "uniform{0..9}" includes 0, so it contributes zero reps (d2_eff = 0.9).
  * geometric "mean 8, capped at 64": support {1, 2, ...} with p = 1/8
    (numpy's geometric), then min(., 64); no zero reps.
  * "uniform{0..2mu}" includes both ends.
  * Bernoulli masks zero the entry with probability 1 - d.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Optional

import numpy as np


@dataclass(frozen=True)
class Config:
    name: str
    case: str  # "a" or "b"
    n: int
    dtype: str  # "float64" / "float32"
    description: str


CONFIGS = {
    "cfg1": Config("cfg1", "a", 256, "float64",
                   "Case-A n=256 fp64: X U[0,1) d1=1; Y U{0..9} d2=1; order-preserving"),
    "cfg2": Config("cfg2", "b", 1024, "float64",
                   "Case-B n=1024 fp64: X U{0..9}*Bern(0.5); Y N(0,1)*Bern(0.5)"),
    "cfg3": Config("cfg3", "a", 4096, "float32",
                   "Case-A n=4096 fp32: X U[-1,1)*Bern(d1), d1 in {0.1,0.5,1}; Y U{0..2mu}, "
                   "mu in {1,4,16}"),
    "cfg4": Config("cfg4", "a", 8192, "float32",
                   "Case-A n=8192 fp32: X U[0,1)*Bern(p_i), p_i~Beta(0.5,0.5); Y geometric "
                   "mean 8 capped at 64"),
    "cfg5": Config("cfg5", "b", 16384, "float32",
                   "Case-B n=16384 fp32: X U{0..31}*Bern(0.9); Y N(0,1)*Bern(0.7)"),
}


def _mask(rng: np.random.Generator, shape, density, dtype) -> np.ndarray:
    return (rng.random(shape, dtype=np.float32) < np.float32(density)).astype(dtype)


def make_inputs(name: str, seed: int = 0, n: Optional[int] = None, d1: float = 1.0,
                mu: int = 1) -> tuple[np.ndarray, np.ndarray]:
    """(lhs, rhs) for BASELINE config `name` (optionally at a smaller n).

    cfg3 takes its sweep point through d1 and mu."""
    cfg = CONFIGS[name]
    n = cfg.n if n is None else int(n)
    dt = np.dtype(cfg.dtype)
    rng = np.random.default_rng(np.random.SeedSequence([1308, 2400, seed, n, int(name[3:])]))
    shape = (n, n)
    if name == "cfg1":
        x = rng.random(shape, dtype=np.float64)
        y = rng.integers(0, 10, shape).astype(np.float64)
    elif name == "cfg2":
        x = rng.integers(0, 10, shape).astype(np.float64) * _mask(rng, shape, 0.5, np.float64)
        y = rng.standard_normal(shape) * _mask(rng, shape, 0.5, np.float64)
    elif name == "cfg3":
        x = (rng.random(shape, dtype=np.float32) * 2.0 - 1.0).astype(np.float32)
        x *= _mask(rng, shape, d1, np.float32)
        y = rng.integers(0, 2 * mu + 1, shape).astype(np.float32)
    elif name == "cfg4":
        p = rng.beta(0.5, 0.5, n).astype(np.float32)
        keep = rng.random(shape, dtype=np.float32) < p[:, None]
        x = rng.random(shape, dtype=np.float32) * keep
        y = np.minimum(rng.geometric(1.0 / 8.0, shape), 64).astype(np.float32)
    elif name == "cfg5":
        x = rng.integers(0, 32, shape, dtype=np.int32).astype(np.float32)
        x *= _mask(rng, shape, 0.9, np.float32)
        y = rng.standard_normal(shape, dtype=np.float32) * _mask(rng, shape, 0.7, np.float32)
    else:
        raise KeyError(name)
    x = np.ascontiguousarray(x, dtype=dt)
    y = np.ascontiguousarray(y, dtype=dt)
    # +0.0 only (the mask can produce -0.0 from negative values times 0)
    x[x == 0] = 0
    y[y == 0] = 0
    return x, y


def expected_additions(case: str, lhs: np.ndarray, rhs: np.ndarray) -> int:
    """Closed-form OpCounts.additions (test_kernels.cpp:45-57, :160-173) with numpy
    integer arithmetic; used to size bench samples and to cross-check counts."""
    if case == "a":
        base_nz = (lhs != 0).astype(np.int64)
        r = np.abs(np.rint(rhs.astype(np.float64))).astype(np.int64).sum(axis=1)
        return int((base_nz.sum(axis=0) * r).sum())
    reps = np.abs(np.rint(lhs.astype(np.float64))).astype(np.int64)
    nnz = (rhs != 0).sum(axis=1).astype(np.int64)
    return int((reps.sum(axis=0) * nnz).sum())


def ladder_additions(case: str, lhs: np.ndarray, rhs: np.ndarray) -> int:
    """FP additions the "fast-ladder" mode PERFORMS on nonzero bases: a term of
    |rep| copies costs floor(log2 |rep|) doublings + popcount(|rep|)
    accumulations (the effective count, expected_additions, charges |rep|)."""
    rep_m = rhs if case == "a" else lhs
    reps = np.abs(np.rint(rep_m.astype(np.float64))).astype(np.int64)
    bits = np.zeros_like(reps)
    top = np.zeros_like(reps)
    r = reps.copy()
    level = 0
    while r.any():
        bits += r & 1
        top = np.where(r != 0, level, top)
        r >>= 1
        level += 1
    cost = np.where(reps != 0, bits + top, 0)
    if case == "a":
        base_nz = (lhs != 0).astype(np.int64)
        return int((base_nz.sum(axis=0) * cost.sum(axis=1)).sum())
    nnz = (rhs != 0).sum(axis=1).astype(np.int64)
    return int((cost.sum(axis=0) * nnz).sum())


def expected_counts(case: str, lhs: np.ndarray, rhs: np.ndarray) -> tuple[int, int, int]:
    """Closed-form OpCounts (additions, multiplications, zero_skips) of valid
    integer-rep operands (SURVEY.md 8.0, test_kernels.cpp:45-57, :160-173):
    Case A zero_skips = #{(i,k): X[i,k] == 0}; Case B zero_skips =
    sum over (i,k) with a nonzero rep of (n - nnz(Y[k,:]))."""
    n = lhs.shape[0]
    adds = expected_additions(case, lhs, rhs)
    if case == "a":
        return adds, 0, int((lhs == 0).sum())
    rep_nz = (np.rint(lhs.astype(np.float64)) != 0).astype(np.int64)
    nnz = (rhs != 0).sum(axis=1).astype(np.int64)
    return adds, 0, int((rep_nz.sum(axis=0) * (n - nnz)).sum())
