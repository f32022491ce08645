"""Compare B-form kernel shapes (dev tool): kernel time and bit-identity.

  python tools/shape_time.py [--variants auto,wide,ring] [--big] [--sweep]

For each BASELINE point (cfg2, cfg3 d1 in {1.0, 0.5} x mu in {1, 4, 16}, cfg4,
cfg5 with --big) every variant (AFMM_BFORM, read at context creation) runs the
same device-resident product; the repeated-addition kernel time (CUDA events
the library records) and the fraction of the measured FP-add peak are printed,
and every variant's Z must equal the first variant's bit for bit (all shapes
are order-preserving). --sweep adds constant-rep dense inputs (rep 1..16).
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1308_2400_b200 as afmm  # noqa: E402
from paper_1308_2400_b200.gen import CONFIGS, make_inputs  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--variants", default="auto,wide,ring")
ap.add_argument("--big", action="store_true")
ap.add_argument("--sweep", action="store_true")
ap.add_argument("--points", default=None, help="comma list like cfg2,cfg3:1.0:1,cfg4")
args = ap.parse_args()
variants = args.variants.split(",")

peak = {"float32": afmm.fp_add_peak(0, "float32")[0], "float64": afmm.fp_add_peak(0, "float64")[0]}
print(f"peak f32 {peak['float32']:.4e} f64 {peak['float64']:.4e}", flush=True)


def run(case, L, R, reps=3):
    res = {}
    ref = None
    for v in variants:
        if v == "auto":
            os.environ.pop("AFMM_BFORM", None)
        else:
            os.environ["AFMM_BFORM"] = v
        ctx = afmm.DeviceContext(0)
        ctx.enable_timing(True)
        O = torch.empty_like(L)
        c = ctx.product(case, L, R, O)
        ks, ts = [], []
        for _ in range(reps):
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record()
            c = ctx.product(case, L, R, O)
            b.record()
            torch.cuda.synchronize()
            ks.append(ctx.last_timing()[1])
            ts.append(a.elapsed_time(b))
        form = ctx.last_form() if case == "a" else "bform"
        ctx.close()
        same = None
        if ref is None:
            ref = O
        else:
            same = bool(torch.equal(O.view(torch.int32) if O.dtype == torch.float32 else
                                    O.view(torch.int64),
                                    ref.view(torch.int32) if ref.dtype == torch.float32 else
                                    ref.view(torch.int64)))
        res[v] = (min(ks), min(ts), c.additions, form, same)
    return res


def show(label, res, dtype):
    parts = []
    for v, (k, t, adds, form, same) in res.items():
        parts.append(f"{v}: k={k:8.3f} step={t:8.3f} ms frac={adds / (k * 1e-3) / peak[dtype]:.3f}"
                     f"{'' if form == 'bform' else ' [' + form + ']'}"
                     f"{'' if same is None else (' same' if same else ' DIFFERENT')}")
    print(f"{label:28s} " + " | ".join(parts), flush=True)


if args.sweep:
    n = 8192
    rng = np.random.default_rng(0)
    Y = torch.from_numpy(rng.standard_normal((n, n), dtype=np.float32)).cuda()
    Y[Y == 0] = 1.0
    for r in (1, 2, 3, 4, 8, 16):
        X = torch.full((n, n), float(r), dtype=torch.float32, device="cuda")
        show(f"dense rep={r}", run("b", X, Y), "float32")
        del X
    del Y

if args.points:
    points = []
    for p in args.points.split(","):
        f = p.split(":")
        points.append((f[0], {} if len(f) == 1 else {"d1": float(f[1]), "mu": int(f[2])}))
else:
    points = [("cfg2", {})] + [("cfg3", {"d1": d, "mu": m}) for d in (1.0, 0.5, 0.1)
                                for m in (1, 4, 16)] + [("cfg4", {})]
    if args.big:
        points.append(("cfg5", {}))
for name, kw in points:
    lhs, rhs = make_inputs(name, seed=0, **kw)
    cfg = CONFIGS[name]
    L = torch.from_numpy(lhs).cuda()
    R = torch.from_numpy(rhs).cuda()
    show(f"{name} {kw}", run(cfg.case, L, R), cfg.dtype)
    del L, R
