"""Device-side seeded generation against the reference's generator.

afmm.generate / DeviceContext.generate run the reference's afmm::generate
(random.hpp:111-129) on the GPU: one std::mt19937_64 stream over the n^2
entries in row-major order, a Bernoulli draw per entry and a value draw per
nonzero entry. The result must be bit-identical to the oracle's restatement
(oracle_generate, itself pinned to the unmodified reference by
tests/test_oracle.py and tests/cpp), for both value roles, edge densities,
seeds across the 64-bit range, sizes that need several chunks of the stream,
and the reference's validation messages (random.hpp:60-79). The device entry
feeds the product directly.
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


CASES = [
    # n, density, mu', integer, low, high
    (1, 1.0, 1.0, True, 0.5, 1.5),
    (2, 0.5, 2.0, True, 0.5, 1.5),
    (7, 0.9, 21.0, True, 0.5, 1.5),
    (33, 0.3, 5.0, True, 0.5, 1.5),
    (256, 1.0, 4.5, False, 0.5, 1.5),  # real role: mu' is not used for values
    (300, 0.7, 1.0, False, -3.0, 2.0),
    (129, 0.0, 3.0, True, 0.5, 1.5),
    (130, 1.0, 1.0, True, 0.5, 1.5),   # mu' = 1: the constant 1
    (64, 0.5, 1.0, False, 2.0, 2.0),   # degenerate bounds
    (1000, 0.25, 9.0, True, 0.5, 1.5),
]


@pytest.mark.parametrize("case", CASES, ids=[f"n{c[0]}_d{c[1]}_mu{c[2]}_{'int' if c[3] else 'real'}"
                                             for c in CASES])
@pytest.mark.parametrize("seed", [0, 12345, 2**64 - 1])
def test_generate_matches_reference_generator(cuda, oracle, case, seed):
    afmm = _api()
    n, d, mu, integer, lo, hi = case
    z = afmm.generate(n, d, mu, integer, seed, lo, hi)
    want = oracle.generate(n, d, mu, integer, seed, lo, hi)
    assert _bits_equal(z, want)
    z32 = afmm.generate(n, d, mu, integer, seed, lo, hi, dtype=np.float32)
    assert _bits_equal(z32, want.astype(np.float32))


@pytest.mark.parametrize("n,d,mu,integer", [
    (800, 0.9, 16.0, True),     # 1.2M draws: 2 stretches (one tree level, a = 1)
    (1500, 1.0, 2.0, True),     # 4.5M draws: 8 stretches (two levels, partial)
    (4096, 0.9, 16.0, True),    # 3.2e7 draws: 51 stretches (three levels)
    (3000, 0.6, 1.0, False),    # 1.4e7 draws: 23 stretches
    (13000, 1.0, 4.0, True),    # 3.4e8 draws: a full chunk of 512 stretches (five levels) + a second chunk
])
def test_generate_several_stretches_and_chunks(cuda, oracle, n, d, mu, integer):
    """Draws from many parallel stretches of the stream, each started from a
    jump-ahead window (the radix-4 tree of k_mt_jump), and from more than one
    chunk, so the carry (automaton state, entries started) and the chunk's end
    window cross chunk boundaries."""
    afmm = _api()
    z = afmm.generate(n, d, mu, integer, 99)
    want = oracle.generate(n, d, mu, integer, 99)
    bad = np.flatnonzero((z.view(np.uint8) != want.view(np.uint8)).reshape(n, -1).any(axis=1))
    assert bad.size == 0, bad[:10]


@pytest.mark.parametrize("args,msg", [
    ((0, 0.5, 2.0, True), "GeneratorSpec: n must be >= 1"),
    ((4, 1.5, 2.0, True), "GeneratorSpec: density must be in [0, 1]"),
    ((4, -0.1, 2.0, False), "GeneratorSpec: density must be in [0, 1]"),
    ((4, 0.5, 0.0, True), "GeneratorSpec: mu_prime must be positive"),
    ((4, 0.5, 2.5, True), "GeneratorSpec: IntegerValued role requires integer mu_prime >= 1"),
    ((4, 0.5, 0.5, True), "GeneratorSpec: IntegerValued role requires integer mu_prime >= 1"),
])
def test_generate_validation_messages(cuda, args, msg):
    afmm = _api()
    with pytest.raises(afmm.InvalidArgument) as ei:
        afmm.generate(*args, seed=1)
    assert str(ei.value) == msg


def test_generate_invalid_real_bounds(cuda):
    afmm = _api()
    for lo, hi in ((2.0, 1.0), (float("nan"), 1.0), (0.0, float("inf"))):
        with pytest.raises(afmm.InvalidArgument) as ei:
            afmm.generate(4, 0.5, 1.0, False, 1, lo, hi)
        assert str(ei.value) == "GeneratorSpec: invalid value bounds"


def test_generate_on_device_feeds_the_product(cuda, oracle):
    """DeviceContext.generate writes both operands into device tensors (one
    with a padded leading dimension), and the product runs on them without a
    host round trip: the reference's generate + afmm_case_a, bit for bit."""
    import torch

    afmm = _api()
    n = 700
    ctx = afmm.DeviceContext(0)
    X = torch.empty((n, n + 9), dtype=torch.float64, device="cuda")[:, :n]
    Y = torch.empty((n, n + 9), dtype=torch.float64, device="cuda")[:, :n]
    ctx.generate(X, 0.8, 1.0, False, 41)
    ctx.generate(Y, 0.6, 5.0, True, 42)
    Z = torch.empty((n, n), dtype=torch.float64, device="cuda")
    counts = ctx.product("a", X, Y, Z)
    ctx.close()
    x = oracle.generate(n, 0.8, 1.0, False, 41)
    y = oracle.generate(n, 0.6, 5.0, True, 42)
    assert _bits_equal(X.cpu().numpy(), x) and _bits_equal(Y.cpu().numpy(), y)
    z, c = oracle.product_mt("a", x, y, 0, n, 16)
    assert (counts.additions, 0, counts.zero_skips) == c
    assert _bits_equal(Z.cpu().numpy(), z)
