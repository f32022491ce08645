"""Timing of the device-side seeded generation against the reference's
generator (dev tool).

  python tools/gen_time.py [n ...]

For each n: afmm::generate of the reference (oracle/_ref, one host core: the
generator is one sequential std::mt19937_64 stream), the oracle's C
restatement, and the GPU (DeviceContext.generate into device memory, CUDA
events; and the host-buffer entry afmm.generate including the copy back).
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1308_2400_b200 as afmm  # noqa: E402
from oracle.oracle import Oracle, Reference, reference_available  # noqa: E402

ns = [int(a) for a in sys.argv[1:]] or [1024, 4096, 16384]
orc = Oracle()
ref = Reference() if reference_available() else None
ctx = afmm.DeviceContext(0)
for n in ns:
    for d, mu, integer in ((0.9, 16.0, True), (0.7, 1.0, False)):
        X = torch.empty((n, n), dtype=torch.float64, device="cuda")
        ctx.generate(X, d, mu, integer, 5)  # warm-up
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        best = 1e30
        for _ in range(3):
            e0.record()
            ctx.generate(X, d, mu, integer, 5)
            e1.record()
            torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1))
        t0 = time.perf_counter()
        h = afmm.generate(n, d, mu, integer, 5)
        t_host = time.perf_counter() - t0
        line = f"n={n} d={d} {'int mu=%g' % mu if integer else 'real'}: gpu {best:.2f} ms, host entry {t_host * 1e3:.1f} ms"
        if n <= 8192:
            t0 = time.perf_counter()
            o = orc.generate(n, d, mu, integer, 5)
            t_orc = time.perf_counter() - t0
            line += f", oracle {t_orc * 1e3:.1f} ms (exact: {np.array_equal(o.view(np.uint8), h.view(np.uint8))})"
            if ref is not None:
                t0 = time.perf_counter()
                r = ref.generate(n, d, mu, integer, 5)
                t_ref = time.perf_counter() - t0
                line += f", reference {t_ref * 1e3:.1f} ms (x{t_ref * 1e3 / best:.0f} vs gpu)"
        print(line, flush=True)
ctx.close()
