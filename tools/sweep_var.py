"""Synthetic Case-B sweep with VARIABLE reps (uniform 1..2r-1) vs constant (dev tool)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1308_2400_b200 as afmm
n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
peak, mhz = afmm.fp_add_peak(0, "float32")
ctx = afmm.DeviceContext(0); ctx.enable_timing(True)
rng = np.random.default_rng(0)
Y = torch.from_numpy(rng.standard_normal((n, n), dtype=np.float32)).cuda(); Y[Y == 0] = 1.0
O = torch.empty_like(Y)
for r in (2, 8, 16):
    for kind in ("const", "var"):
        if kind == "const":
            X = torch.full((n, n), float(r), dtype=torch.float32, device="cuda")
        else:
            X = torch.from_numpy(rng.integers(1, 2 * r, (n, n)).astype(np.float32)).cuda()
        c = ctx.product("b", X, Y, O)
        ks = []
        for _ in range(3):
            c = ctx.product("b", X, Y, O); ks.append(ctx.last_timing()[1])
        k = min(ks)
        print(f"  {kind:5s} rep~{r:3d} kernel {k:9.3f} ms frac {c.additions / (k * 1e-3) / peak:.3f}", flush=True)
