"""Kernel-efficiency sweep on synthetic Case-B shapes (dev tool).

Dense Y (no zero bases) and a constant rep r isolate the repeated-addition
kernel's instruction efficiency from the structural zero-base waste:
effective adds/s / peak should approach 1 for large r.

  [AFMM_BFORM=wide|ring|small|tmem|mr] [AFMM_LIB=...] python tools/sweep.py [n]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1308_2400_b200 as afmm  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
peak, mhz = afmm.fp_add_peak(0, "float32")
ctx = afmm.DeviceContext(0)
ctx.enable_timing(True)
rng = np.random.default_rng(0)
Y = torch.from_numpy(rng.standard_normal((n, n), dtype=np.float32)).cuda()
Y[Y == 0] = 1.0
O = torch.empty_like(Y)
print(f"variant={os.environ.get('AFMM_BFORM', 'auto')} n={n} peak={peak:.4e} @ {mhz:.0f} MHz")
for r in (1, 2, 4, 8, 16, 32):
    X = torch.full((n, n), float(r), dtype=torch.float32, device="cuda")
    for _ in range(2):
        c = ctx.product("b", X, Y, O)
    kms = []
    for _ in range(3):
        c = ctx.product("b", X, Y, O)
        kms.append(ctx.last_timing()[1])
    k = min(kms)
    rate = c.additions / (k * 1e-3)
    print(f"  rep={r:3d} kernel {k:9.3f} ms  {rate:.4e} adds/s  frac {rate / peak:.3f}", flush=True)
ctx.close()
