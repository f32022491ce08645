"""Reference-facing call with PAGEABLE host buffers (numpy arrays, like a
std::vector-backed DenseMatrix) against page-locked ones, and the staged copy
pipeline's worker count (dev tool; output kept in profiles/r02/pageable/).

  python tools/pageable_time.py            # pageable vs pinned, default workers
  python tools/pageable_time.py workers    # pageable, AFMM_STAGE_WORKERS = 1, 2, 4, 6, 8
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1308_2400_b200 as afmm  # noqa: E402
from paper_1308_2400_b200.gen import make_inputs  # noqa: E402

sweep = len(sys.argv) > 1 and sys.argv[1] == "workers"
for name, n in (("cfg5", 16384), ("cfg5", 8192), ("cfg4", 8192), ("cfg3", 4096)):
    lhs, rhs = make_inputs(name, seed=0, n=n)
    case = "a" if name in ("cfg4", "cfg3") else "b"
    fn = afmm.afmm_case_a if case == "a" else afmm.afmm_case_b
    out = np.empty_like(lhs)
    runs = []
    if sweep:
        runs = [(f"pageable workers={w}", lhs, rhs, out, w) for w in ("1", "2", "4", "6", "8")]
    else:
        hl, hr = torch.from_numpy(lhs).pin_memory(), torch.from_numpy(rhs).pin_memory()
        hz = torch.empty_like(hl).pin_memory()
        runs = [("pageable", lhs, rhs, out, None), ("pinned", hl.numpy(), hr.numpy(), hz.numpy(), None)]
    for label, a, b, o, w in runs:
        if w:
            os.environ["AFMM_STAGE_WORKERS"] = w
        ts = []
        for _ in range(3):
            t0 = time.perf_counter()
            r = fn(a, b, out=o, timing=True)
            ts.append((time.perf_counter() - t0) * 1e3)
        print(f"{name} n={n} {lhs.dtype} {label}: wall ms {['%.1f' % t for t in ts]} "
              f"device total {r.timing['total_ms']:.1f} compute {r.timing['compute_ms']:.1f}",
              flush=True)
