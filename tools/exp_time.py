"""Compact timing of one library build (dev tool for kernel experiments).

  AFMM_LIB=build/exp/<name>/libafmm_b200.so python tools/exp_time.py [--big]

Prints the repeated-addition kernel's fraction of the measured FP-add peak on
constant-rep dense inputs (rep 1, 2, 4, 16) and the whole-product time of
cfg2, cfg3 (d1=1, mu=1/4/16) and cfg4 (and cfg5 with --big, cfg3 d1 = 0.1 with --aform).
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1308_2400_b200 as afmm  # noqa: E402
from paper_1308_2400_b200.gen import CONFIGS, make_inputs  # noqa: E402

peak32, mhz = afmm.fp_add_peak(0, "float32")
ctx = afmm.DeviceContext(0)
ctx.enable_timing(True)
lib = os.environ.get("AFMM_LIB", "in-tree")
out = [f"lib={lib.split('/')[-2] if '/' in lib else lib} peak={peak32:.4e}@{mhz:.0f}MHz"]

n = 8192
rng = np.random.default_rng(0)
Y = torch.from_numpy(rng.standard_normal((n, n), dtype=np.float32)).cuda()
Y[Y == 0] = 1.0
O = torch.empty_like(Y)
for r in (1, 2, 4, 16):
    X = torch.full((n, n), float(r), dtype=torch.float32, device="cuda")
    ctx.product("b", X, Y, O)
    ks = []
    for _ in range(3):
        c = ctx.product("b", X, Y, O)
        ks.append(ctx.last_timing()[1])
    out.append(f"r{r}={c.additions / (min(ks) * 1e-3) / peak32:.3f}")
del X, Y, O

points = [("cfg2", {}), ("cfg3", {"d1": 1.0, "mu": 1}), ("cfg3", {"d1": 1.0, "mu": 4}),
          ("cfg3", {"d1": 1.0, "mu": 16}), ("cfg4", {})]
if "--aform" in sys.argv:  # sparse-X points that run the A-form kernel
    points += [("cfg3", {"d1": 0.1, "mu": m}) for m in (1, 4, 16)]
if "--big" in sys.argv:
    points.append(("cfg5", {}))
for name, kw in points:
    lhs, rhs = make_inputs(name, seed=0, **kw)
    L = torch.from_numpy(lhs).cuda()
    R = torch.from_numpy(rhs).cuda()
    O = torch.empty_like(L)
    case = CONFIGS[name].case
    ctx.product(case, L, R, O)
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    ms = []
    for _ in range(3):
        a.record()
        ctx.product(case, L, R, O, sync=False)
        b.record()
        ctx.finish()
        torch.cuda.synchronize()
        ms.append(a.elapsed_time(b))
    tag = name + ("".join(f"_{k}{v}" for k, v in kw.items()) if kw else "")
    out.append(f"{tag}={min(ms):.3f}ms")
    del L, R, O
print(" ".join(out), flush=True)
ctx.close()
