"""Quick device-resident timing of the product at BASELINE shapes (dev tool)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1308_2400_b200 as afmm  # noqa: E402
from paper_1308_2400_b200.gen import CONFIGS, expected_additions, make_inputs  # noqa: E402


def time_cfg(name, reps=3, **kw):
    cfg = CONFIGS[name]
    t0 = time.time()
    lhs, rhs = make_inputs(name, seed=0, **kw)
    tgen = time.time() - t0
    ctx = afmm.DeviceContext(0)
    L = torch.from_numpy(lhs).cuda()
    R = torch.from_numpy(rhs).cuda()
    O = torch.empty_like(L)
    counts = ctx.product(cfg.case, L, R, O)  # warm-up
    torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    ms = []
    for _ in range(reps):
        a.record()
        ctx.product(cfg.case, L, R, O, sync=False)
        b.record()
        ctx.finish()
        torch.cuda.synchronize()
        ms.append(a.elapsed_time(b))
    best = min(ms)
    rate = counts.additions / (best * 1e-3)
    print(f"{name} {kw} n={cfg.n} adds={counts.additions:.4e} (closed form "
          f"{expected_additions(cfg.case, lhs, rhs):.4e}) best {best:.3f} ms -> {rate:.4e} adds/s "
          f"(gen {tgen:.1f}s)", flush=True)
    ctx.close()
    return rate


if __name__ == "__main__":
    peak32, mhz = afmm.fp_add_peak(0, "float32")
    peak64, mhz64 = afmm.fp_add_peak(0, "float64")
    print(f"peak f32 {peak32:.4e} adds/s @ {mhz:.0f} MHz; f64 {peak64:.4e} @ {mhz64:.0f} MHz")
    which = sys.argv[1:] or ["cfg1", "cfg2", "cfg3", "cfg4", "cfg5"]
    for name in which:
        if name == "cfg3":
            for d1 in (0.1, 0.5, 1.0):
                for mu in (1, 4, 16):
                    r = time_cfg("cfg3", d1=d1, mu=mu)
                    print(f"   frac of f32 peak {r / peak32:.3f}")
        else:
            r = time_cfg(name)
            pk = peak64 if CONFIGS[name].dtype == "float64" else peak32
            print(f"   frac of peak {r / pk:.3f}")
