"""Single-process multi-GPU product behind the C ABI (afmm_options.num_devices).

The pool gives one GPU per call, so the shards run as several contexts on
cuda:0 (options.devices = [0, 0, ...]: a device may be listed more than once);
every step of the multi-device path -- chunked host->device copies from
parallel host threads, per-shard validation, the peer completion of Y and the
per-k vector, the merged statuses, the cut by predicted time, the peer copies
of the missing X rows, the per-shard product straight into `out` -- runs, with
same-device copies standing in for NVLink. Results must be bit-identical to the
single-device product and the oracle for every shard count, and errors must be
the reference's first offender over the whole operands.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _bits_equal(a, b):
    a = np.ascontiguousarray(a)
    b = np.ascontiguousarray(b)
    return a.shape == b.shape and np.array_equal(a.view(np.uint8), b.view(np.uint8))


def _api():
    import paper_1308_2400_b200 as afmm

    return afmm


@pytest.mark.parametrize("case,name,n,dt,shards,partition", [
    ("a", "cfg1", 256, np.float64, 2, "work"),
    ("b", "cfg2", 1024, np.float64, 2, "work"),
    ("b", "cfg5", 777, np.float32, 3, "work"),
    ("a", "cfg4", 1100, np.float32, 2, "work"),
    ("a", "cfg4", 1100, np.float64, 3, "rows"),
    ("a", "cfg3", 1300, np.float32, 4, "work"),
    ("b", "cfg5", 5, np.float32, 3, "work"),
    ("a", "cfg1", 2, np.float64, 3, "rows"),
])
def test_multi_device_host_call_bit_exact(cuda, oracle, case, name, n, dt, shards, partition):
    from paper_1308_2400_b200.gen import make_inputs

    afmm = _api()
    kw = {"d1": 0.1, "mu": 4} if name == "cfg3" else {}
    lhs, rhs = make_inputs(name, seed=31, n=n, **kw)
    lhs, rhs = lhs.astype(dt), rhs.astype(dt)
    fn = afmm.afmm_case_a if case == "a" else afmm.afmm_case_b
    one = fn(lhs, rhs)
    res = fn(lhs, rhs, devices=[0] * shards, partition=partition, timing=True)
    z, c = oracle.product_mt(case, lhs, rhs, 0, n, 16)
    assert (res.counts.additions, res.counts.multiplications, res.counts.zero_skips) == c
    assert _bits_equal(res.product, z)
    assert _bits_equal(res.product, one.product)
    assert res.timing["devices"] == shards and res.timing["total_ms"] > 0.0


@pytest.mark.parametrize("dt", [np.float32, np.float64])
def test_multi_device_pinned_out_zero_copy(cuda, oracle, dt):
    """Case B into page-locked `out`: every shard's kernels store their Z rows
    straight into the caller's buffer; untouched when validation fails."""
    import torch

    from paper_1308_2400_b200.gen import make_inputs

    afmm = _api()
    n = 1030
    lhs, rhs = make_inputs("cfg5", seed=3, n=n)
    lhs, rhs = lhs.astype(dt), rhs.astype(dt)
    tdt = torch.float32 if dt == np.float32 else torch.float64
    out = torch.full((n, n), 7.0, dtype=tdt).pin_memory().numpy()
    res = afmm.afmm_case_b(lhs, rhs, out=out, devices=[0, 0])
    z, c, _ = oracle.product("b", lhs, rhs)
    assert (res.counts.additions, 0, res.counts.zero_skips) == c
    assert _bits_equal(out, z)
    out[:] = 7.0
    bad = lhs.copy()
    bad[n - 3, 5] = 0.5  # in the second shard's rows
    with pytest.raises(afmm.DomainError, match=rf"lhs\[{n - 3}\]\[5\] = 0.500000 is not"):
        afmm.afmm_case_b(bad, rhs, out=out, devices=[0, 0])
    assert np.all(out == 7.0)


@pytest.mark.parametrize("case", ["a", "b"])
def test_multi_device_errors_are_the_global_first_offender(cuda, case):
    """Each shard validates its own chunk of both operands; the merged status
    reports the reference's error: non-finite elements first (DenseMatrix
    construction, matrix.hpp:31-35), then the rep operand's first offender in
    row-major order over the WHOLE matrix (kernels.hpp:25-43)."""
    afmm = _api()
    n = 600
    rng = np.random.default_rng(2)
    bases = rng.standard_normal((n, n))
    reps = rng.integers(-5, 6, (n, n)).astype(np.float64)
    if case == "a":
        lhs, rhs, repm, opname = bases, reps, "rhs", "rhs"
    else:
        lhs, rhs, repm, opname = reps, bases, "lhs", "lhs"
    r = (rhs if case == "a" else lhs).copy()
    r[450, 7] = 2.5      # third shard's chunk
    r[220, 3] = -0.75    # second shard's chunk: the first offender
    args = (lhs, r) if case == "a" else (r, rhs)
    fn = afmm.afmm_case_a if case == "a" else afmm.afmm_case_b
    with pytest.raises(afmm.DomainError,
                       match=rf"afmm_case_{case}: {opname}\[220\]\[3\] = -0.750000 is not "
                             r"integer-valued"):
        fn(*args, devices=[0, 0, 0])
    big = (rhs if case == "a" else lhs).copy()
    big[500, 1] = 2.0 ** 60
    args = (lhs, big) if case == "a" else (big, rhs)
    with pytest.raises(afmm.DomainError, match=r"\[500\]\[1\] exceeds the exact integer range"):
        fn(*args, devices=[0, 0])
    # a non-finite base in the last shard beats a rep error in the first
    nb = (lhs if case == "a" else rhs).copy()
    nb[599, 0] = np.inf
    r2 = (rhs if case == "a" else lhs).copy()
    r2[0, 0] = 0.5
    args = (nb, r2) if case == "a" else (r2, nb)
    with pytest.raises(afmm.DomainError, match="non-finite"):
        fn(*args, devices=[0, 0, 0])
    # and a valid call right after is exact on every shard
    args = (lhs, rhs)
    a = fn(*args, devices=[0, 0, 0])
    b = fn(*args)
    assert _bits_equal(a.product, b.product) and a.counts == b.counts


def test_multi_device_invalid_options(cuda):
    afmm = _api()
    with pytest.raises(afmm.InvalidArgument):
        afmm.afmm_case_a(np.eye(3), np.eye(3), devices=[0, 99])
    with pytest.raises(afmm.InvalidArgument):
        afmm.afmm_case_a(np.eye(3), np.eye(3), devices=[])


def test_multi_device_case_a_cut_follows_predicted_time(cuda, oracle):
    """Case A rows sorted by density (Beta(0.5, 0.5) densities, cfg4): the cut
    by predicted time differs from the equal-row cut, and both are exact."""
    afmm = _api()
    from paper_1308_2400_b200.gen import make_inputs

    n = 2100
    lhs, rhs = make_inputs("cfg4", seed=8, n=n)
    order = np.argsort((lhs != 0).sum(axis=1), kind="stable")
    lhs = np.ascontiguousarray(lhs[order])
    z, c = oracle.product_mt("a", lhs, rhs, 0, n, 16)
    for partition in ("work", "rows"):
        res = afmm.afmm_case_a(lhs, rhs, devices=[0, 0, 0, 0], partition=partition)
        assert _bits_equal(res.product, z), partition
        assert res.counts.additions == c[0]


def test_bench_single_process_multi_gpu_path_runs(cuda):
    """`python bench.py --gpus 2` without torchrun: one process drives both
    shards (here both on cuda:0: AFMM_SINGLE_DEVICE, a functional run) and
    reports n_gpus = 2."""
    import json
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, AFMM_SINGLE_DEVICE="1")
    cmd = [sys.executable, os.path.join(root, "bench.py"), "--gpus", "2", "--steps", "2",
           "--warmup", "3", "--size", "1024", "--no-cpu-baseline"]
    r = subprocess.run(cmd, cwd=root, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["e2e"]["value"] > 0
    assert "one process" in d["config"]["parallelism"]
    assert d["config"]["test_mode"].startswith("AFMM_SINGLE_DEVICE")
    assert d["gpu_launches"] > 0
