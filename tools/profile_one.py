"""One device-resident AFMM product of a BASELINE config (the command profiled by ncu).

  python tools/profile_one.py cfg5 [--d1 1.0 --mu 16] [--reps 1]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1308_2400_b200 as afmm  # noqa: E402
from paper_1308_2400_b200.gen import CONFIGS, make_inputs  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("config")
p.add_argument("--d1", type=float, default=1.0)
p.add_argument("--mu", type=int, default=16)
p.add_argument("--n", type=int, default=None)
p.add_argument("--reps", type=int, default=1)
p.add_argument("--mode", default="order-preserving", choices=["order-preserving", "fast", "fast-ladder"])
a = p.parse_args()
cfg = CONFIGS[a.config]
lhs, rhs = make_inputs(a.config, seed=0, n=a.n, d1=a.d1, mu=a.mu)
L = torch.from_numpy(lhs).cuda()
R = torch.from_numpy(rhs).cuda()
O = torch.empty_like(L)
ctx = afmm.DeviceContext(0)
ctx.enable_timing(True)
for _ in range(a.reps):
    c = ctx.product(cfg.case, L, R, O, mode=a.mode)
    print(a.config, c, "kernel", ctx.last_form(), "phases ms (prepass, kernel, epilogue):",
          ctx.last_timing(), flush=True)
ctx.close()
