"""Row-sharded multi-GPU AFMM product (one process per GPU, torch.distributed/NCCL).

Z row i depends only on X row i and all of Y (kernels.hpp:119 and :148 loop over
independent rows), so the product shards by contiguous Z-row ranges:

  1. every rank computes the same row cuts on its own GPU (afmm_partition_device;
     Y and X are replicated, so no communication): equal W_i for Case B, equal
     modeled kernel time for Case A, whose A-form time follows a row's nonzero
     bases and whose B-form time does not;
  2. every rank runs the product on its row slab (afmm_product_device);
  3. the slabs land in rank 0's Z. Default ("p2p"): rank 0 exports its Z
     buffer over CUDA IPC, the other ranks map it (peer access over NVLink /
     NVSwitch) and their repeated-addition kernels store Z tiles straight into
     it as they finish, so the transfer overlaps the compute and there is no
     gather step; the ranks then meet at one barrier. Fallback ("sendrecv",
     or when the buffer cannot be exported): one batched point-to-point
     exchange after the compute (NCCL send/recv; NCCL has no variable-size
     gather). AFMM_GATHER=sendrecv forces the fallback.

Results are bit-identical for every world size: each Z element is computed by
exactly one rank with the same per-element add sequence.
"""
from __future__ import annotations

import os
from typing import Optional

import numpy as np
import torch

from .afmm import DeviceContext, OpCounts, RawRows, ipc_close, ipc_export, ipc_open


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


class PeerResult:
    """Rank 0's result buffer as seen from every rank (CUDA IPC).

    Each call broadcasts rank 0's (handle, offset, leading dimension) -- 81
    bytes -- so all ranks agree on the target even if the caller changes
    buffers between calls; a rank re-maps only when the handle changes. A
    zero flag byte means rank 0 could not export (the caller falls back to
    send/recv)."""

    def __init__(self, dist, rank: int, device: int):
        self.dist, self.rank, self.device = dist, rank, device
        self._key = None
        self._ptr = None

    def exchange(self, z_full):
        """(enabled, pointer of rank 0's Z in this process or None on rank 0, its ld).

        Every rank must be able to map the buffer: a rank that cannot (no peer
        access, IPC blocked) says so in an all-reduced flag and then ALL ranks
        fall back to the send/recv gather together (none is left waiting in a
        barrier the others never reach)."""
        msg = np.zeros(81, dtype=np.uint8)
        if self.rank == 0 and getattr(z_full, "is_cuda", False):
            try:
                handle, offset = ipc_export(z_full)
                msg[0] = 1
                msg[1:65] = np.frombuffer(handle, dtype=np.uint8)
                msg[65:81] = np.frombuffer(np.array([offset, z_full.stride(0)],
                                                    dtype=np.uint64).tobytes(), dtype=np.uint8)
            except Exception:
                msg[0] = 0
        on_gpu = self.dist.get_backend() == "nccl"
        t = torch.from_numpy(msg)
        if on_gpu:
            t = t.cuda(self.device)
        self.dist.broadcast(t, src=0)
        msg = t.cpu().numpy()
        ok, ptr, ld = False, None, 0
        if msg[0] != 0:
            offset, ld = (int(v) for v in np.frombuffer(msg[65:81].tobytes(), dtype=np.uint64))
            ok = True
            if self.rank != 0:
                key = msg[:73].tobytes()
                if key != self._key:
                    self.close()
                    try:
                        self._ptr = ipc_open(self.device, msg[1:65].tobytes(), offset)
                        self._key = key
                    except Exception:
                        ok = False
                ptr = self._ptr
        flag = torch.tensor([1 if ok else 0], dtype=torch.int32,
                            device=f"cuda:{self.device}" if on_gpu else "cpu")
        self.dist.all_reduce(flag, op=self.dist.ReduceOp.MIN)
        if int(flag.item()) == 0:
            return False, None, 0
        return True, ptr, ld

    def close(self) -> None:
        if self._ptr is not None:
            ipc_close(self._ptr)
        self._ptr, self._key = None, None


class ShardedProduct:
    """One rank's share of a row-sharded product on device-resident operands."""

    def __init__(self, ctx: DeviceContext, dist, rank: int, world: int,
                 gather: Optional[str] = None):
        self.ctx = ctx
        self.dist = dist
        self.rank = rank
        self.world = world
        self.cuts: Optional[np.ndarray] = None
        # "p2p": kernels store into rank 0's Z over CUDA IPC; "sendrecv": NCCL
        # gather after the compute; "none": each rank keeps its slab (rows
        # cuts[rank]..cuts[rank+1] in slab_buf), e.g. to copy it to its host
        self.gather = gather or os.environ.get("AFMM_GATHER", "p2p")
        self.used_p2p = False
        self._peer = PeerResult(dist, rank, getattr(ctx, "device", 0)) if world > 1 and \
            self.gather == "p2p" else None

    def run(self, case: str, lhs, rhs, z_full, slab_buf,
            mode: str = "order-preserving") -> OpCounts:
        """lhs, rhs: full n x n device tensors on every rank; z_full: n x n on rank 0;
        slab_buf: a scratch n x n tensor on ranks > 0. Returns this rank's counts."""
        n = lhs.shape[0]
        if self.world == 1:
            counts = self.ctx.product(case, lhs, rhs, z_full, 0, n, mode=mode)
            self.cuts = np.array([0, n])
            return counts
        cuts = self.ctx.partition(case, lhs, rhs, self.world)
        self.cuts = cuts
        r0, r1 = int(cuts[self.rank]), int(cuts[self.rank + 1])
        if self.gather == "none":
            return self.ctx.product(case, lhs, rhs, slab_buf[: max(r1 - r0, 1)], r0, r1,
                                    mode=mode)
        ok, peer, ld = self._peer.exchange(z_full) if self._peer else (False, None, 0)
        self.used_p2p = ok
        if ok:
            # every slab is written in place into rank 0's Z (peer stores from
            # the kernels); the barrier orders them before rank 0's reads
            if self.rank == 0:
                out = z_full[r0:r1]
            else:
                out = RawRows(peer, ld, str(lhs.dtype).replace("torch.", ""), n).rows(r0)
            counts = self.ctx.product(case, lhs, rhs, out, r0, r1, mode=mode)
            self.dist.barrier()
            return counts
        out = z_full[r0:r1] if self.rank == 0 else slab_buf[: max(r1 - r0, 1)]
        counts = self.ctx.product(case, lhs, rhs, out, r0, r1, mode=mode)
        gather_rows(self.dist, z_full, out[: r1 - r0], cuts, self.rank, self.world)
        return counts

    def close(self) -> None:
        """Unmap rank 0's result buffer (p2p mode)."""
        if self._peer:
            self._peer.close()
