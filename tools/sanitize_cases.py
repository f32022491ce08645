"""The smallest product of every kernel path, for compute-sanitizer runs.

  compute-sanitizer --tool memcheck|racecheck|synccheck|initcheck --error-exitcode 99 \\
      python tools/sanitize_cases.py

Each case is checked bit for bit against the CPU oracle (so a run that the
tool lets finish also proves the result), and covers one path of the library:
the three B-form tile shapes (Case B and Case A on transposed operands), the
A-form, the device-side row split, the reassociated fast mode (split-k +
reduce), CUDA-graph replays, a validation error (kernels exit early), the
zero-copy page-locked output, the multi-device host path (several shards
on one device: chunked copies, peer completion, cut, per-shard product), and
the small-rep group kernel (both cases and a split).
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1308_2400_b200 as afmm  # noqa: E402
from oracle.oracle import Oracle  # noqa: E402
from paper_1308_2400_b200.gen import make_inputs  # noqa: E402

oracle = Oracle()
done = []


def check(label, case, lhs, rhs, z, counts=None):
    want, c, _ = oracle.product(case, lhs, rhs)
    assert np.array_equal(np.ascontiguousarray(z).view(np.uint8), want.view(np.uint8)), label
    if counts is not None:
        assert (counts.additions, counts.multiplications, counts.zero_skips) == c, label
    done.append(label)


def device(label, case, lhs, rhs, variant=None, mode="order-preserving", reps=1):
    if variant:
        os.environ["AFMM_BFORM"] = variant
    else:
        os.environ.pop("AFMM_BFORM", None)
    ctx = afmm.DeviceContext(0)
    L = torch.from_numpy(lhs).cuda()
    R = torch.from_numpy(rhs).cuda()
    O = torch.empty_like(L)
    for _ in range(reps):
        c = ctx.product(case, L, R, O, mode=mode)
    z = O.cpu().numpy()
    ctx.close()
    if mode in ("fast", "fast-ladder"):
        want, cc, _ = oracle.product(case, lhs.astype(np.float64), rhs.astype(np.float64))
        err = np.abs(z - want).max() / max(1.0, np.abs(want).max())
        assert err < 1e-4, (label, err)
        done.append(label)
        return
    check(label, case, lhs, rhs, z, c)


l1, r1 = make_inputs("cfg1", seed=1, n=96)
l2, r2 = make_inputs("cfg2", seed=1, n=200)
l5, r5 = make_inputs("cfg5", seed=1, n=300)
for v in ("wide", "ring", "small"):
    device(f"case B fp64 {v}", "b", l2, r2, v)
    device(f"case B fp32 {v}", "b", l5, r5, v)
    device(f"case A fp64 {v}", "a", l1, r1, v)
la, ra = make_inputs("cfg3", seed=1, n=1100, d1=0.1, mu=4)
device("case A A-form (device choice)", "a", la, ra)
l4, r4 = make_inputs("cfg4", seed=1, n=1100)
device("case A split (forced)", "a", l4, r4, "hybrid")
device("case A fp32 fast mode", "a", l4, r4, mode="fast")
device("case B fp64 fast mode", "b", l2, r2, mode="fast")
device("case A fp32 fast-ladder mode", "a", l4, r4, mode="fast-ladder")
device("case B fp32 fast-ladder mode", "b", l5, r5, mode="fast-ladder")
device("case B graph replays", "b", l2, r2, reps=4)
device("case A graph replays", "a", la, ra, reps=4)
# the small-rep group kernel (every rep in 0..2): Case A (column groups, ragged
# tiles), Case B (row groups), and the split with a group B part
lg, rg = make_inputs("cfg3", seed=1, n=777, d1=1.0, mu=1)
device("case A group kernel", "a", lg, rg)
device("case B group kernel", "b", rg.T.copy(), lg)
lh, rh = make_inputs("cfg3", seed=2, n=1100, d1=0.5, mu=1)
device("case A split with group B part (forced)", "a", lh, rh, "hybrid")
os.environ.pop("AFMM_BFORM", None)

# packed 4-byte list entries (n >= 2048, every |rep| <= 127), both cases, and
# the int2 lists at the same size (AFMM_BFORM=nopack)
lp, rp = make_inputs("cfg3", seed=3, n=2048, d1=0.5, mu=4)
device("case A packed lists", "a", lp, rp)
device("case B packed lists", "b", rp.T.copy(), lp)
device("case B int2 lists at n = 2048", "b", rp.T.copy(), lp, "nopack")
os.environ.pop("AFMM_BFORM", None)

bad = l2.copy()
bad[7, 3] = 0.5
try:
    afmm.afmm_case_b(bad, r2)
    raise AssertionError("no error")
except afmm.DomainError:
    done.append("validation error")

pinned = torch.empty((300, 300), dtype=torch.float32).pin_memory().numpy()
res = afmm.afmm_case_b(l5, r5, out=pinned)
check("zero-copy pinned output", "b", l5, r5, pinned, res.counts)
res = afmm.afmm_case_a(l4, r4, devices=[0, 0, 0])
check("multi-device host path (3 shards)", "a", l4, r4, res.product, res.counts)
res = afmm.afmm_case_b(l5, r5, devices=[0, 0])
check("multi-device host path (2 shards)", "b", l5, r5, res.product, res.counts)
print(f"sanitize cases: {len(done)} paths exact:", "; ".join(done), flush=True)
