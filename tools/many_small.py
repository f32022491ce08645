"""Throughput of many independent small products (dev tool): one DeviceContext
per CUDA stream, all enqueued before any is awaited, vs one after another.

  python tools/many_small.py [config] [count]
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1308_2400_b200 as afmm  # noqa: E402
from paper_1308_2400_b200.gen import CONFIGS, make_inputs  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg1"
count = int(sys.argv[2]) if len(sys.argv) > 2 else 32
cfg = CONFIGS[name]
ins = []
for i in range(count):
    lhs, rhs = make_inputs(name, seed=i)
    L, R = torch.from_numpy(lhs).cuda(), torch.from_numpy(rhs).cuda()
    ins.append((L, R, torch.empty_like(L)))
streams = [torch.cuda.Stream() for _ in range(count)]
ctxs = [afmm.DeviceContext(0) for _ in range(count)]
for c, s in zip(ctxs, streams):
    c.set_stream(s)
adds = 0
for c, (L, R, O) in zip(ctxs, ins):  # warm-up (allocations, attributes)
    adds += c.product(cfg.case, L, R, O).additions
torch.cuda.synchronize()
for rnd in range(3):
    t0 = time.perf_counter()
    for c, (L, R, O) in zip(ctxs, ins):
        c.product(cfg.case, L, R, O)
    seq = time.perf_counter() - t0
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for c, (L, R, O) in zip(ctxs, ins):
        c.product(cfg.case, L, R, O, sync=False)
    for c in ctxs:
        c.finish()
    conc = time.perf_counter() - t0
    print(f"{name} x{count}: sequential {seq * 1e3:.2f} ms ({adds / seq:.3e} adds/s), "
          f"concurrent streams {conc * 1e3:.2f} ms ({adds / conc:.3e} adds/s)", flush=True)
for c in ctxs:
    c.close()
