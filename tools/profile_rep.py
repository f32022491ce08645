"""One Case-B product with a constant rep on dense random bases (ncu target).

  python tools/profile_rep.py REP [N]
"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1308_2400_b200 as afmm
r = int(sys.argv[1]); n = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
rng = np.random.default_rng(0)
Y = torch.from_numpy(rng.standard_normal((n, n), dtype=np.float32)).cuda(); Y[Y == 0] = 1.0
X = torch.full((n, n), float(r), dtype=torch.float32, device="cuda")
O = torch.empty_like(Y)
ctx = afmm.DeviceContext(0); ctx.enable_timing(True)
c = ctx.product("b", X, Y, O)
print("rep", r, "n", n, c, "kernel ms", ctx.last_timing()[1])
