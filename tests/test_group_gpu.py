"""The small-rep group kernel (k_bgroup) against the reference order.

When every rep of the product is in 0..2 (fp32, order-preserving mode) the
device chooses k_bgroup for the B-form part: five B-form rows per warp share
each staged base row, and one jump-table dispatch per k replaces five rep
loops (bform.cu, tools/gen_jumptable.py). The choice is made on the device
from the validated rep statistics, so these tests check both sides of it --
the kernel is bit-identical to the oracle (the reference's per-element add
order) and counts are the closed forms; any rep outside 0..2, a negative rep,
fp64, the fast mode or a forced k_bform shape keeps k_bform -- across ragged
sizes, row slabs, the Case A split, graph replays that change the decision,
multi-device shards and the output-sentinel frame.
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


def _bases(rng, n, density=0.7, dt=np.float32):
    b = (rng.standard_normal((n, n)) * (rng.random((n, n)) < density)).astype(dt)
    b[rng.random((n, n)) < 0.02] = -0.0  # signed zeros stay bit-neutral
    return b


def _reps(rng, n, hi=2, density=0.8, dt=np.float32):
    return (rng.integers(0, hi + 1, (n, n)) * (rng.random((n, n)) < density)).astype(dt)


def _run(ctx, case, lhs, rhs, r0=0, r1=None, **kw):
    import torch

    n = lhs.shape[0]
    r1 = n if r1 is None else r1
    L = torch.from_numpy(lhs).cuda()
    R = torch.from_numpy(rhs).cuda()
    O = torch.full((max(r1 - r0, 1), n), 3.0, dtype=L.dtype, device="cuda")
    counts = ctx.product(case, L, R, O, r0, r1, **kw)
    return O[: r1 - r0].cpu().numpy(), counts


@pytest.mark.parametrize("case,n", [("b", 1000), ("b", 1537), ("b", 3), ("a", 1280), ("a", 777),
                                    ("a", 2049)])
def test_group_kernel_bit_exact(cuda, oracle, case, n):
    """Ragged n (groups of 5 rows and 512-column tiles both partial), both
    cases, reps in {0, 1, 2}: k_bgroup runs and matches the oracle bit for bit."""
    afmm = _api()
    rng = np.random.default_rng(n)
    bases, reps = _bases(rng, n), _reps(rng, n)
    lhs, rhs = (bases, reps) if case == "a" else (reps, bases)
    ctx = afmm.DeviceContext(0)
    z, counts = _run(ctx, case, lhs, rhs)
    form = ctx.last_form()
    ctx.close()
    assert form in ("group", "split-group"), form
    zo, c = oracle.product_mt(case, lhs, rhs, 0, n, 16)
    assert (counts.additions, 0, counts.zero_skips) == c
    assert _bits_equal(z, zo)


@pytest.mark.parametrize("d1", [1.0, 0.5])
def test_group_kernel_cfg3_mu1(cuda, oracle, d1):
    """cfg3's mu = 1 points (Y uniform {0, 1, 2}) at n = 1536 pick the group
    kernel through the device-side Case A choice."""
    from paper_1308_2400_b200.gen import make_inputs

    afmm = _api()
    lhs, rhs = make_inputs("cfg3", seed=3, n=1536, d1=d1, mu=1)
    ctx = afmm.DeviceContext(0)
    z, counts = _run(ctx, "a", lhs, rhs)
    assert ctx.last_form() == "group"
    ctx.close()
    zo, c = oracle.product_mt("a", lhs, rhs, 0, 1536, 16)
    assert (counts.additions, 0, counts.zero_skips) == c
    assert _bits_equal(z, zo)


@pytest.mark.parametrize("what", ["rep3", "negative", "fp64", "fast", "nogroup", "wide"])
def test_group_kernel_fallbacks(cuda, oracle, monkeypatch, what):
    """Outside the group kernel's domain k_bform runs, with the same bits."""
    afmm = _api()
    rng = np.random.default_rng(7)
    n = 900
    dt = np.float64 if what == "fp64" else np.float32
    bases, reps = _bases(rng, n, dt=dt), _reps(rng, n, dt=dt)
    if what == "rep3":
        reps[n - 1, n - 1] = 3.0
    if what == "negative":
        reps[n // 2, 7] = -1.0
    if what in ("nogroup", "wide"):
        monkeypatch.setenv("AFMM_BFORM", what)
    mode = "fast" if what == "fast" else "order-preserving"
    ctx = afmm.DeviceContext(0)
    for case, lhs, rhs in (("b", reps, bases), ("a", bases, reps)):
        z, counts = _run(ctx, case, lhs, rhs, mode=mode)
        assert ctx.last_form() == "bform", (what, case)
        zo, c = oracle.product_mt(case, lhs, rhs, 0, n, 16)
        assert (counts.additions, 0, counts.zero_skips) == c
        if mode == "fast":
            continue
        assert _bits_equal(z, zo), (what, case)
    ctx.close()


def test_group_kernel_row_slabs_and_padded_ld(cuda, oracle):
    """Device API: Case B row slabs whose length is not a multiple of 5 and
    whose start is not group-aligned, with padded and unaligned leading
    dimensions (the base operand is copied to an aligned buffer)."""
    import torch

    afmm = _api()
    rng = np.random.default_rng(12)
    n = 611
    bases, reps = _bases(rng, n), _reps(rng, n)
    ctx = afmm.DeviceContext(0)
    for case, lhs, rhs in (("b", reps, bases), ("a", bases, reps)):
        zfull, _ = oracle.product_mt(case, lhs, rhs, 0, n, 16)
        for ld in (n, n + 3, 640):
            L = torch.zeros((n, ld), dtype=torch.float32, device="cuda")
            R = torch.zeros((n, ld), dtype=torch.float32, device="cuda")
            L[:, :n] = torch.from_numpy(lhs)
            R[:, :n] = torch.from_numpy(rhs)
            for r0, r1 in ((0, n), (3, 139), (606, 611), (200, 201)):
                O = torch.full((r1 - r0, ld), 9.0, dtype=torch.float32, device="cuda")
                counts = ctx.product(case, L[:, :n], R[:, :n], O[:, :n], r0, r1)
                assert ctx.last_form() == "group", (case, ld, r0, r1)
                _, c = oracle.product_mt(case, lhs, rhs, r0, r1, 16)
                assert (counts.additions, 0, counts.zero_skips) == c
                assert _bits_equal(O[:, :n].cpu().numpy(), zfull[r0:r1]), (case, ld, r0, r1)
    ctx.close()


def test_group_kernel_in_case_a_split(cuda, oracle, monkeypatch):
    """Case A with Beta(0.5, 0.5) row densities and reps in {0, 1, 2}, split
    forced: the sparsest rows in the A-form, the rest through k_bgroup over the
    gathered X^T columns (dyn_ncols); bit-exact."""
    afmm = _api()
    monkeypatch.setenv("AFMM_BFORM", "hybrid")
    rng = np.random.default_rng(41)
    n = 1300
    p = rng.beta(0.5, 0.5, n)
    x = (rng.random((n, n)) * (rng.random((n, n)) < p[:, None])).astype(np.float32)
    y = _reps(rng, n, density=1.0)
    ctx = afmm.DeviceContext(0)
    z, counts = _run(ctx, "a", x, y)
    assert ctx.last_form() == "split-group"
    ctx.close()
    zo, c = oracle.product_mt("a", x, y, 0, n, 16)
    assert (counts.additions, 0, counts.zero_skips) == c
    assert _bits_equal(z, zo)


def test_group_decision_replayed_graphs(cuda, oracle):
    """Repeated identical device calls replay a CUDA graph; the group decision
    is on the device, so raising one rep to 3 in place switches the replay to
    k_bform (and back), bit-exact every time, with a constant launch count."""
    import torch

    afmm = _api()
    rng = np.random.default_rng(5)
    n = 700
    bases, reps = _bases(rng, n), _reps(rng, n)
    ctx = afmm.DeviceContext(0)
    L = torch.from_numpy(reps).cuda()
    R = torch.from_numpy(bases).cuda()
    O = torch.empty_like(L)
    forms, launches = [], []
    for it in range(6):
        cur = reps.copy()
        if it in (3, 4):
            cur[11, 13] = 3.0
        L.copy_(torch.from_numpy(cur))
        k0 = afmm.kernel_launch_count()
        assert ctx.product("b", L, R, O, sync=False) is None
        c = ctx.finish()
        launches.append(afmm.kernel_launch_count() - k0)
        forms.append(ctx.last_form())
        zo, cc = oracle.product_mt("b", cur, bases, 0, n, 16)
        assert (c.additions, 0, c.zero_skips) == cc, it
        assert _bits_equal(O.cpu().numpy(), zo), (it, forms[-1])
    ctx.close()
    assert forms == ["group"] * 3 + ["bform"] * 2 + ["group"], forms
    assert len(set(launches[1:])) == 1, launches


@pytest.mark.parametrize("case", ["a", "b"])
def test_group_kernel_multi_device(cuda, oracle, case):
    """The multi-device host call (3 shards on one GPU): each shard's status
    is seeded with the merged rep statistics (validation ran per chunk), so
    every shard picks the group kernel; bit-identical to one device."""
    afmm = _api()
    rng = np.random.default_rng(17)
    n = 1111
    bases, reps = _bases(rng, n), _reps(rng, n)
    lhs, rhs = (bases, reps) if case == "a" else (reps, bases)
    fn = afmm.afmm_case_a if case == "a" else afmm.afmm_case_b
    one = fn(lhs, rhs)
    res = fn(lhs, rhs, devices=[0, 0, 0], timing=True)
    zo, c = oracle.product_mt(case, lhs, rhs, 0, n, 16)
    assert (res.counts.additions, res.counts.multiplications, res.counts.zero_skips) == c
    assert _bits_equal(res.product, zo)
    assert _bits_equal(one.product, zo)
    assert res.timing["form"] in ("group", "split-group"), res.timing


def test_group_kernel_writes_only_its_output(cuda, oracle):
    """Sentinel frame around the output view (offset rows / columns, padded
    ld): every byte outside it survives the group kernel, both cases."""
    import torch

    afmm = _api()
    rng = np.random.default_rng(61)
    n = 1030
    bases, reps = _bases(rng, n), _reps(rng, n)
    sentinel = -12345.5
    ctx = afmm.DeviceContext(0)
    for case, lhs, rhs in (("a", bases, reps), ("b", reps, bases)):
        L = torch.from_numpy(lhs).cuda()
        R = torch.from_numpy(rhs).cuda()
        r0, r1 = 17, n - 5
        big = torch.full((r1 - r0 + 9, n + 40), sentinel, dtype=torch.float32, device="cuda")
        view = big[4:4 + r1 - r0, 16:16 + n]
        ctx.product(case, L, R, view, r0, r1)
        assert ctx.last_form() == "group", case
        b = big.cpu().numpy()
        inside = np.zeros(b.shape, dtype=bool)
        inside[4:4 + r1 - r0, 16:16 + n] = True
        assert np.all(b[~inside] == sentinel), case
        z, _ = oracle.product_mt(case, lhs, rhs, r0, r1, 16)
        assert _bits_equal(b[4:4 + r1 - r0, 16:16 + n], z), case
    ctx.close()
