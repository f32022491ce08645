"""Row-sharded multi-GPU AFMM product (one process per GPU, torch.distributed/NCCL).

Z row i depends only on X row i and all of Y (kernels.hpp:119 and :148 loop over
independent rows), so the product shards by contiguous Z-row ranges:

  1. every rank computes the exact per-row work W_i on its own GPU
     (afmm_row_work_device; Y and X are replicated, so no communication) and
     cuts the rows into `world` ranges of equal total work (afmm_partition_rows);
  2. every rank runs the product on its row slab (afmm_product_device);
  3. the slabs are gathered into rank 0's Z with one batched point-to-point
     exchange over NVLink (NCCL send/recv; NCCL has no variable-size gather),
     the only collective of the path.

Results are bit-identical for every world size: each Z element is computed by
exactly one rank with the same per-element add sequence.
"""
from __future__ import annotations

from typing import Optional

import numpy as np
import torch

from .afmm import DeviceContext, OpCounts, partition_rows


def gather_rows(dist, z_full, slab, cuts, rank: int, world: int) -> None:
    """Collect row slabs into rank 0's `z_full` (rank 0's own slab is already in place).

    `slab` is this rank's (cuts[rank+1]-cuts[rank]) x n block; `z_full` is the
    n x n result on rank 0 (ignored elsewhere)."""
    # gloo has no CUDA point-to-point: stage device slabs through host memory
    # (the functional multi-rank test on one GPU; the bench uses NCCL)
    staged = dist.get_backend() == "gloo" and getattr(z_full, "is_cuda", False)
    ops, landing = [], []
    if rank == 0:
        for r in range(1, world):
            r0, r1 = int(cuts[r]), int(cuts[r + 1])
            if r1 > r0:
                dst = z_full[r0:r1]
                if staged:
                    buf = torch.empty(dst.shape, dtype=dst.dtype)
                    landing.append((dst, buf))
                    dst = buf
                ops.append(dist.P2POp(dist.irecv, dst, r))
    else:
        if int(cuts[rank + 1]) > int(cuts[rank]):
            ops.append(dist.P2POp(dist.isend, slab.cpu() if staged else slab, 0))
    if ops:
        for req in dist.batch_isend_irecv(ops):
            req.wait()
    for dst, buf in landing:
        dst.copy_(buf)


class ShardedProduct:
    """One rank's share of a row-sharded product on device-resident operands."""

    def __init__(self, ctx: DeviceContext, dist, rank: int, world: int):
        self.ctx = ctx
        self.dist = dist
        self.rank = rank
        self.world = world
        self.cuts: Optional[np.ndarray] = None

    def run(self, case: str, lhs, rhs, z_full, slab_buf,
            mode: str = "order-preserving") -> OpCounts:
        """lhs, rhs: full n x n device tensors on every rank; z_full: n x n on rank 0;
        slab_buf: a scratch n x n tensor on ranks > 0. Returns this rank's counts."""
        n = lhs.shape[0]
        if self.world == 1:
            counts = self.ctx.product(case, lhs, rhs, z_full, 0, n, mode=mode)
            self.cuts = np.array([0, n])
            return counts
        work = self.ctx.row_work(case, lhs, rhs)
        cuts = partition_rows(work, self.world)
        self.cuts = cuts
        r0, r1 = int(cuts[self.rank]), int(cuts[self.rank + 1])
        out = z_full[r0:r1] if self.rank == 0 else slab_buf[: max(r1 - r0, 1)]
        counts = self.ctx.product(case, lhs, rhs, out, r0, r1, mode=mode)
        gather_rows(self.dist, z_full, out[: r1 - r0], cuts, self.rank, self.world)
        return counts
