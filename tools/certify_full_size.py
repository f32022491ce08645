"""Full-size parity certificate: every row of every BASELINE configuration.

  python tools/certify_full_size.py [--configs cfg5,cfg4,...] > certificate.log

For each configuration at its BASELINE size (cfg1, cfg2, the 9 cfg3 points,
cfg4, cfg5) the product is computed on the GPU (device-resident operands,
order-preserving mode, the automatic kernel choice) and EVERY row of Z is
compared bit for bit with the vectorised CPU checker (oracle/fast_check.c,
itself pinned to the scalar oracle and the unmodified reference by
tests/test_oracle.py); the counts are compared with the closed forms. One line
per configuration: sizes, additions, kernel form, rows checked, mismatching
rows, and the SHA-256 of Z (so two runs can be compared without the data).
Exit code 1 on any mismatch.
"""
import argparse
import hashlib
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1308_2400_b200 as afmm  # noqa: E402
from oracle.oracle import FastCheck  # noqa: E402
from paper_1308_2400_b200.gen import CONFIGS, expected_counts, make_inputs  # noqa: E402

ALL = ["cfg1", "cfg2"] + [f"cfg3:{d}:{m}" for d in (0.1, 0.5, 1.0) for m in (1, 4, 16)] + \
    ["cfg4", "cfg5"]

ap = argparse.ArgumentParser()
ap.add_argument("--configs", default=",".join(ALL))
ap.add_argument("--seed", type=int, default=0)
args = ap.parse_args()

fc = FastCheck()
print(f"# full-size certificate, seed {args.seed}, host threads {os.cpu_count()}, "
      f"GPU {torch.cuda.get_device_name(0)}", flush=True)
failed = 0
for spec in args.configs.split(","):
    f = spec.split(":")
    name = f[0]
    kw = {} if len(f) == 1 else {"d1": float(f[1]), "mu": int(f[2])}
    cfg = CONFIGS[name]
    lhs, rhs = make_inputs(name, seed=args.seed, **kw)
    ctx = afmm.DeviceContext(0)
    L = torch.from_numpy(lhs).cuda()
    R = torch.from_numpy(rhs).cuda()
    O = torch.empty_like(L)
    t0 = time.time()
    c = ctx.product(cfg.case, L, R, O)
    torch.cuda.synchronize()
    t_gpu = time.time() - t0
    form = ctx.last_form()
    ctx.close()
    z = O.cpu().numpy()
    del L, R, O
    t0 = time.time()
    want = fc.product(cfg.case, lhs, rhs)
    t_cpu = time.time() - t0
    rows_bad = np.flatnonzero((z.view(np.uint8) != want.view(np.uint8))
                              .reshape(z.shape[0], -1).any(axis=1))
    counts_ok = (c.additions, c.multiplications, c.zero_skips) == expected_counts(cfg.case, lhs,
                                                                                  rhs)
    ok = rows_bad.size == 0 and counts_ok
    failed += 0 if ok else 1
    print(f"{'OK  ' if ok else 'FAIL'} {spec:14s} case {cfg.case} n={cfg.n} {cfg.dtype} "
          f"adds={c.additions} zero_skips={c.zero_skips} form={form} rows_checked={z.shape[0]} "
          f"rows_mismatch={rows_bad.size} counts={'closed-form' if counts_ok else 'WRONG'} "
          f"sha256(Z)={hashlib.sha256(z.tobytes()).hexdigest()[:32]} "
          f"gpu_s={t_gpu:.2f} check_s={t_cpu:.1f}", flush=True)
print(f"# {'all configurations bit-exact on every row' if not failed else f'{failed} FAILED'}")
sys.exit(1 if failed else 0)
