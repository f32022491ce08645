#!/usr/bin/env python
"""bench.py -- effective additions/sec of the B200 AFMM product (BASELINE.json metric).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg5] [--impl b200|reference]

A step is one AFMM product over the workload's synthetic operands (BASELINE.json
config; default cfg5 = Case-B n=16384 fp32, ~4.3e13 additions, the config the
metric's 1/2/4/8-GPU scaling is specified on). Under torchrun each rank owns one
GPU; the rows are partitioned by work and every rank's kernels store its Z rows
straight into rank 0's result (CUDA IPC peer mapping over NVLink) inside the step.

  value  adds/s with operands resident in HBM (CUDA events, max over ranks)
  e2e    the same metric through the reference-facing C-ABI call with pinned HOST
         buffers (H2D of X and Y + product + D2H of Z inside the timed region)
  roofline  the repeated-addition kernel's effective adds/s (per-launch CUDA events
         around k_bform on its stream) against the MEASURED CUDA-core FP-add peak
         (afmm_fp_add_peak microbenchmark, same process, same GPU)
  cpu_baseline  the oracle port (bit-identical to the reference, tests/test_oracle.py)
         on the host cores over a stated row sample

--impl reference times the reference's CPU algorithm (the oracle port, all host
threads) on a bounded row sample of the same workload, rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "effective additions/sec (sum |rep| over nonzero bases)"
UNIT = "adds/s"


def parse_args():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=5)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="b200", choices=["b200", "reference"])
    p.add_argument("--config", default="cfg5", choices=["cfg1", "cfg2", "cfg3", "cfg4", "cfg5"])
    p.add_argument("--d1", type=float, default=1.0, help="cfg3 sweep point")
    p.add_argument("--mu", type=int, default=16, help="cfg3 sweep point")
    p.add_argument("--seed", type=int, default=0)
    p.add_argument("--size", dest="n", type=int, default=None,
                   help="reduced problem size (tests only; the config's n by default)")
    p.add_argument("--mode", default="order-preserving", choices=["order-preserving", "fast", "fast-ladder"],
                   help="order-preserving = bit-exact with the reference (default); fast = "
                        "reassociated split-k within 1e-12/1e-5")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-secondary", action="store_true",
                   help="skip the other BASELINE configurations' device-resident numbers")
    p.add_argument("--cpu-seconds", type=float, default=12.0,
                   help="target CPU time of one baseline sample")
    return p.parse_args()


# ---------------------------------------------------------------------------
# clocks during the timed region (NVML)
# ---------------------------------------------------------------------------

_REASONS = {
    0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
    0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
    0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting",
}


class ClockSampler(threading.Thread):
    def __init__(self, device: int, period: float = 0.1):
        super().__init__(daemon=True)
        self.device = device
        # NVML enumerates by PCI bus, CUDA may not (CUDA_VISIBLE_DEVICES,
        # CUDA_DEVICE_ORDER): identify the device by its PCI address
        try:
            import torch

            pr = torch.cuda.get_device_properties(device)
            self.pci = f"{pr.pci_domain_id:08x}:{pr.pci_bus_id:02x}:{pr.pci_device_id:02x}.0"
        except Exception:
            self.pci = None
        self.period = period
        self.samples = []
        self.reasons = set()
        self.max_mhz = None
        self._halt = threading.Event()
        self.ok = False

    def run(self):
        try:
            import pynvml

            pynvml.nvmlInit()
            h = None
            if self.pci:
                try:
                    h = pynvml.nvmlDeviceGetHandleByPciBusId(self.pci.encode())
                except Exception:
                    h = None
            if h is None:
                h = pynvml.nvmlDeviceGetHandleByIndex(self.device)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
            self.ok = True
            while not self._halt.is_set():
                self.samples.append(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM))
                try:
                    mask = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                except Exception:
                    mask = pynvml.nvmlDeviceGetCurrentClocksThrottleReasons(h)
                for bit, name in _REASONS.items():
                    if mask & bit and bit != 0x1:
                        self.reasons.add(name)
                time.sleep(self.period)
        except Exception as e:  # NVML missing: report, do not fail the bench
            self.error = repr(e)

    def stop(self):
        self._halt.set()
        self.join(timeout=2)
        return {
            "sm_mhz": statistics.median(self.samples) if self.samples else None,
            "sm_max_mhz": self.max_mhz,
            "reasons": sorted(self.reasons),
            "samples": len(self.samples),
        }


# ---------------------------------------------------------------------------
# CPU baseline: the reference's CPU path (unmodified kernels) on a row sample
# ---------------------------------------------------------------------------

class CpuBaseline:
    """The reference's CPU path on the host cores, on a bounded row sample.

    kind "reference": the UNMODIFIED afmm_case_{a,b} (oracle/_ref/libafmm_ref.so,
    built from /root/reference in the build container; fp32 inputs widened
    exactly to the reference's fp64), one call per thread, each on the lhs with
    only its block of rows kept (rows are independent, kernels.hpp:119,148).
    The per-call overhead of the n x n call (allocation, validation, zero-row
    scans) is measured by the same batch with empty blocks and subtracted.
    kind "port": the oracle restatement (bit-identical, tests/test_oracle.py),
    used only when the reference library is absent."""

    def __init__(self, case, lhs, rhs, threads):
        from oracle.oracle import Oracle, Reference, reference_available

        self.case = case
        self.n = lhs.shape[0]
        self.kind = "reference" if reference_available() else "port"
        if self.kind == "reference":
            # each concurrent reference call holds two n x n fp64 matrices (its
            # masked lhs and the product); stay within half the available RAM
            try:
                avail = os.sysconf("SC_AVPHYS_PAGES") * os.sysconf("SC_PAGE_SIZE")
            except (ValueError, OSError):
                avail = 0
            per_call = 2 * 8 * self.n * self.n
            if avail > 0:
                threads = min(threads, max(1, int(0.5 * avail // per_call)))
        self.threads = max(1, min(threads, self.n))
        if self.kind == "reference":
            self.ref = Reference()
            self.lhs = np.ascontiguousarray(lhs, dtype=np.float64)
            self.rhs = np.ascontiguousarray(rhs, dtype=np.float64)
            self.overhead, _, _ = self.ref.rows_batch(case, self.lhs, self.rhs,
                                                      [(0, 0)] * self.threads)
        else:
            self.oracle = Oracle()
            self.lhs, self.rhs = lhs, rhs
            self.overhead = 0.0

    def _blocks(self, b):
        starts = np.linspace(0, self.n - b, self.threads).astype(int)
        return [(int(st), int(st) + b) for st in starts]

    def batch(self, b):
        """b rows per thread -> (work seconds, additions)."""
        if self.kind == "reference":
            wall, adds, _ = self.ref.rows_batch(self.case, self.lhs, self.rhs, self._blocks(b))
            return max(wall - self.overhead, 1e-6), adds
        t0 = time.perf_counter()
        adds = 0
        for r0, r1 in self._blocks(b):
            _, c = self.oracle.product_mt(self.case, self.lhs, self.rhs, r0, r1, self.threads)
            adds += c[0]
        return time.perf_counter() - t0, adds

    def rows_for(self, target_s):
        """Rows per thread for about target_s seconds of work."""
        secs, _ = self.batch(1)
        return int(max(1, min(self.n // self.threads, round(target_s / max(secs, 1e-4)))))

    def describe(self, b, adds, secs):
        what = ("unmodified reference afmm_case_%s (oracle/_ref/libafmm_ref.so, fp64; fp32 "
                "inputs widened exactly), one call per thread on its row block, per-call "
                "overhead %.2f s (measured with empty blocks) subtracted"
                % (self.case, self.overhead)) if self.kind == "reference" else \
            "oracle/afmm_oracle.c restatement (bit-identical to the unmodified reference)"
        return (f"{self.threads} threads x {b} rows ({self.threads * b} of {self.n} rows, blocks "
                f"spread evenly), {adds:.4e} additions in {secs:.1f} s; {what}")


def run_reference_arm(args, rank):
    """--impl reference: the reference's own CPU implementation of the path (unmodified
    afmm_case_{a,b} from oracle/_ref) on all host threads, rank 0 only."""
    if rank != 0:
        return
    from paper_1308_2400_b200.gen import CONFIGS, make_inputs

    cfg = CONFIGS[args.config]
    lhs, rhs = make_inputs(args.config, seed=args.seed, n=args.n, d1=args.d1, mu=args.mu)
    cpu = CpuBaseline(cfg.case, lhs, rhs, os.cpu_count() or 1)
    b = cpu.rows_for(args.cpu_seconds * 0.5)
    for _ in range(max(0, min(args.warmup, 1))):
        cpu.batch(1)
    adds = 0
    secs = 0.0
    for _ in range(args.steps):
        s_, a = cpu.batch(b)
        adds += a
        secs += s_
    value = adds / secs
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * secs / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f64 (the reference is fp64-only; fp32 configs widened exactly)"
        if cfg.dtype == "float32" else "f64",
        "data": "synthetic (seeded numpy, BASELINE.json distributions)",
        "config": _config_dict(args, cfg),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cpu.threads, "kind": cpu.kind,
                         "sample": "per step: " + cpu.describe(b, adds // args.steps,
                                                               secs / args.steps)},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def _config_dict(args, cfg):
    n = args.n or cfg.n
    d = {"workload": f"{cfg.name}: {cfg.description}"
                     + ("" if n == cfg.n else f" [REDUCED to n={n}: test run, not the config]"),
         "case": cfg.case, "n": n,
         "mode": "order-preserving (bit-exact)" if args.mode == "order-preserving"
         else "fast (reassociated split-k, tolerance 1e-12 f64 / 1e-5 f32)" if args.mode == "fast"
         else "fast-ladder (fast + each term's |rep| copies summed as a doubling ladder: "
              "floor(log2 rep) + popcount(rep) adds per term; the metric still counts |rep|)",
         "parallelism": f"row-partition x{args.gpus}" + (
             " (one process per GPU, torchrun)" if int(os.environ.get("WORLD_SIZE", "1")) > 1
             else " (one process, all GPUs)" if args.gpus > 1 else ""),
         "l2": "operands larger than L2" if n >= 4096 else "L2 flushed between steps"}
    if cfg.name == "cfg3":
        d["d1"] = args.d1
        d["mu"] = args.mu
    return d


# ---------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------

def refuse(why):
    """No JSON line for a run that would not measure what it says."""
    print(f"bench.py: refusing to report: {why}", file=sys.stderr, flush=True)
    sys.exit(2)


def main():
    args = parse_args()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference_arm(args, rank)
        return
    if world > 1 and args.gpus != world:
        refuse(f"--gpus {args.gpus} under torchrun with WORLD_SIZE={world}")
    if world == 1 and args.gpus > 1:
        run_single_process(args)
        return

    import torch
    import torch.distributed as dist

    import paper_1308_2400_b200 as afmm
    from paper_1308_2400_b200.distributed import ShardedProduct, gather_rows
    from paper_1308_2400_b200.gen import CONFIGS, make_inputs

    # AFMM_DIST_BACKEND=gloo + AFMM_SINGLE_DEVICE=1: functional test of the N > 1
    # path with every rank on cuda:0 (tests/test_multirank_gpu.py); never a
    # measurement. The bench proper is one process per GPU over NCCL.
    backend = os.environ.get("AFMM_DIST_BACKEND", "nccl")
    if os.environ.get("AFMM_SINGLE_DEVICE"):
        local = 0
    torch.cuda.set_device(local)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
        dist.barrier()
    red_dev = "cpu" if backend != "nccl" else None
    cfg = CONFIGS[args.config]
    tdt = torch.float32 if cfg.dtype == "float32" else torch.float64
    es = 4 if cfg.dtype == "float32" else 8

    lhs, rhs = make_inputs(args.config, seed=args.seed, n=args.n, d1=args.d1, mu=args.mu)
    n = lhs.shape[0]
    dev = torch.device("cuda", local)
    L = torch.from_numpy(lhs).to(dev)
    R = torch.from_numpy(rhs).to(dev)
    Z = torch.empty((n, n), dtype=tdt, device=dev)  # rank 0: full result; others: slab scratch
    ctx = afmm.DeviceContext(local)
    ctx.enable_timing(True)
    sharded = ShardedProduct(ctx, dist if world > 1 else None, rank, world)
    peak, peak_mhz = afmm.fp_add_peak(local, cfg.dtype)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev) if n < 4096 else None

    def barrier():
        if world > 1:
            dist.barrier()

    def step():
        return sharded.run(cfg.case, L, R, Z, Z, mode=args.mode)

    for _ in range(args.warmup):
        counts = step()
    torch.cuda.synchronize()

    # ---- device-resident timed loop ----
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    sampler = ClockSampler(local)
    sampler.start()
    launches0 = afmm.kernel_launch_count()
    barrier()
    torch.cuda.synchronize()
    total_ms = 0.0
    kernel_ms = []
    rank_adds = 0
    for _ in range(args.steps):
        if flush is not None:
            flush.fill_(1.0)  # evict the operands from L2 between steps (untimed)
            torch.cuda.synchronize()
        e0.record()
        counts = step()
        e1.record()
        torch.cuda.synchronize()
        total_ms += e0.elapsed_time(e1)
        kernel_ms.append(ctx.last_timing()[1])
        rank_adds = counts.additions
    torch.cuda.synchronize()
    barrier()
    launches = afmm.kernel_launch_count() - launches0
    clocks = sampler.stop()

    t = torch.tensor([total_ms, float(rank_adds)], dtype=torch.float64, device=red_dev or dev)
    if world > 1:
        tmax = t.clone()
        dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
        tsum = t.clone()
        dist.all_reduce(tsum, op=dist.ReduceOp.SUM)
        total_ms = float(tmax[0])
        job_adds = int(tsum[1])
    else:
        job_adds = rank_adds
    ms_per_step = total_ms / args.steps
    value = job_adds / (ms_per_step * 1e-3)

    # ---- roofline of the repeated-addition kernel (this rank's launch) ----
    kms = statistics.median(kernel_ms)
    if not kms > 0.0:
        raise RuntimeError(f"no device timing of the repeated-addition kernel: {kernel_ms}")
    achieved = rank_adds / (kms * 1e-3)
    traffic = _ncu_traffic(args.config if args.config != "cfg3"
                           else f"cfg3_d{args.d1:g}_mu{args.mu}")
    form = ctx.last_form()
    roofline = {
        "bound": "fp-add",
        "bound_detail": "CUDA-core FP add issue (FADD2/DADD; FADD under predicates in the "
                        "A-form): no tensor cores (they would multiply), far right of the HBM "
                        "ridge",
        "kernel": afmm.FORM_KERNELS.get(form, "k_bform"),
        "achieved": achieved / 1e12, "peak": peak / 1e12, "unit": "TFLOP/s",
        "unit_note": "FLOP = one FP add (fp32 FADD2 lanes / fp64 DADD); the kernel does no "
                     "multiplications, so FP-add/s is its FLOP/s",
        "frac": achieved / peak,
        "peak_source": f"measured in-process by afmm_fp_add_peak ({'FADD2' if es == 4 else 'DADD'}"
                       f" chains) at {peak_mhz:.0f} MHz",
        "algorithmic_units_per_launch": rank_adds,
        "kernel_ms": kms,
        "step_share": kms / ms_per_step if world == 1 else None,
        "traffic": traffic,
        "hbm_check": _hbm_check(traffic),
    }

    # ---- end to end through the reference-facing API ----
    e2e = None
    if not args.no_e2e:
        e2e = _e2e(args, afmm, dist, torch, world, rank, local, cfg, lhs, rhs, es, job_adds,
                   sharded, L, R, Z)

    # ---- the other BASELINE configurations (device-resident, this GPU) ----
    secondary = None
    if rank == 0 and world == 1 and not args.no_secondary and args.n is None:
        secondary = _secondary(args, afmm, torch, local, {"float32": peak} if es == 4 else {})

    # ---- the headline configuration in the reassociated modes ----
    reassoc = None
    if rank == 0 and world == 1 and not args.no_secondary and args.mode == "order-preserving":
        reassoc = _reassociated(args, afmm, torch, ctx, cfg, lhs, rhs, L, R, Z, peak)

    # ---- CPU baseline ----
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        base = CpuBaseline(cfg.case, lhs, rhs, os.cpu_count() or 1)
        b = base.rows_for(args.cpu_seconds)
        secs, adds = base.batch(b)
        cpu = {"value": adds / secs, "unit": UNIT, "cores": base.threads, "kind": base.kind,
               "sample": base.describe(b, adds, secs)}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f32" if es == 4 else "f64",
            "data": "synthetic (seeded numpy PCG64, BASELINE.json distributions; no dataset)",
            "config": _config_dict(args, cfg),
            "frac_of_fp_add_peak": value / (peak * world),
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
            "gpu_launches": launches, "clocks": clocks,
        }
        if args.mode == "fast-ladder":
            # the metric counts the additions the product stands for (sum |rep|);
            # the ladder performs fewer -- report those too, and the pipe
            # fraction they amount to
            from paper_1308_2400_b200.gen import ladder_additions
            performed = ladder_additions(cfg.case, lhs, rhs)
            line["performed_additions"] = performed
            line["effective_over_performed"] = job_adds / max(performed, 1)
            if world == 1:
                line["performed_frac_of_fp_add_peak"] = performed / (kms * 1e-3) / peak
        if secondary is not None:
            line["secondary_configs"] = secondary
        if reassoc is not None:
            line["reassociated_modes"] = reassoc
        if world > 1:
            line["config"]["gather"] = (
                "in-kernel peer stores into rank 0's Z (CUDA IPC mapping, NVLink), one barrier"
                if sharded.used_p2p else "NCCL send/recv of the Z slabs after the compute")
        print(json.dumps(line), flush=True)
    sharded.close()
    ctx.close()
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def run_single_process(args):
    """--gpus G without torchrun: one process drives G GPUs.

    value: device-resident operands replicated on every GPU; the rows are cut
    by predicted kernel time (afmm_row_cost_device) and each GPU's kernels
    store its Z rows straight into GPU 0's Z over NVLink (peer access), all
    enqueued asynchronously; the step time is the max over GPUs of CUDA events
    on each GPU's stream.
    e2e: the reference-facing C-ABI call with host buffers and
    options.num_devices = G (afmm_case_*(..., devices=[0..G-1])): chunked H2D,
    NVLink completion of Y, per-GPU products, Z rows straight to host."""
    import torch

    import paper_1308_2400_b200 as afmm
    from paper_1308_2400_b200.afmm import RawRows
    from paper_1308_2400_b200.gen import CONFIGS, make_inputs

    G = args.gpus
    # AFMM_SINGLE_DEVICE=1: functional test with every shard on cuda:0
    # (tests/test_multirank_gpu.py), never a measurement
    single = bool(os.environ.get("AFMM_SINGLE_DEVICE"))
    dev = [0 if single else g for g in range(G)]
    if not single and torch.cuda.device_count() < G:
        refuse(f"--gpus {G} but only {torch.cuda.device_count()} CUDA devices are visible")
    cfg = CONFIGS[args.config]
    tdt = torch.float32 if cfg.dtype == "float32" else torch.float64
    es = 4 if cfg.dtype == "float32" else 8
    lhs, rhs = make_inputs(args.config, seed=args.seed, n=args.n, d1=args.d1, mu=args.mu)
    n = lhs.shape[0]
    Ls = [torch.from_numpy(lhs).to(f"cuda:{dev[g]}") for g in range(G)]
    Rs = [torch.from_numpy(rhs).to(f"cuda:{dev[g]}") for g in range(G)]
    Z = torch.empty((n, n), dtype=tdt, device="cuda:0")
    ctxs = [afmm.DeviceContext(dev[g]) for g in range(G)]
    for c in ctxs:
        c.enable_timing(True)
    peak, peak_mhz = afmm.fp_add_peak(0, cfg.dtype)
    cost = ctxs[0].row_cost(cfg.case, Ls[0], Rs[0])
    cuts = afmm.partition_rows(cost, G)
    zrows = RawRows(Z.data_ptr(), Z.stride(0), cfg.dtype, n, n)
    flush = [torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=f"cuda:{d}")
             for d in sorted(set(dev))] if n < 4096 else None
    devices = sorted(set(dev))

    def step():
        for g in range(G):
            r0, r1 = int(cuts[g]), int(cuts[g + 1])
            with torch.cuda.device(dev[g]):
                ctxs[g].product(cfg.case, Ls[g], Rs[g], zrows.rows(r0), r0, r1, sync=False,
                                mode=args.mode)
        return [c.finish() for c in ctxs]

    for _ in range(args.warmup):
        step()
    for d in devices:
        torch.cuda.synchronize(d)
    sampler = ClockSampler(0)
    sampler.start()
    launches0 = afmm.kernel_launch_count()
    total_ms = 0.0
    kernel_ms = []
    adds = 0
    for _ in range(args.steps):
        if flush is not None:
            for f in flush:
                f.fill_(1.0)
        for d in devices:
            torch.cuda.synchronize(d)
        ev = []
        for d in devices:
            with torch.cuda.device(d):
                a = torch.cuda.Event(enable_timing=True)
                b = torch.cuda.Event(enable_timing=True)
                a.record()
                ev.append((a, b))
        counts = step()
        for i, d in enumerate(devices):
            with torch.cuda.device(d):
                ev[i][1].record()
        for d in devices:
            torch.cuda.synchronize(d)
        total_ms += max(a.elapsed_time(b) for a, b in ev)
        kernel_ms.append(ctxs[0].last_timing()[1])
        adds = sum(c.additions for c in counts)
    launches = afmm.kernel_launch_count() - launches0
    clocks = sampler.stop()
    ms_per_step = total_ms / args.steps
    value = adds / (ms_per_step * 1e-3)
    kms = statistics.median(kernel_ms)
    rank0_adds = int(counts[0].additions)
    roofline = {
        "bound": "fp-add", "kernel": afmm.FORM_KERNELS.get(ctxs[0].last_form(), "k_bform"),
        "achieved": rank0_adds / (kms * 1e-3) / 1e12, "peak": peak / 1e12, "unit": "TFLOP/s",
        "unit_note": "FLOP = one FP add; GPU 0's repeated-addition kernel on its row share",
        "frac": rank0_adds / (kms * 1e-3) / peak,
        "peak_source": f"measured in-process by afmm_fp_add_peak at {peak_mhz:.0f} MHz",
        "algorithmic_units_per_launch": rank0_adds, "kernel_ms": kms, "traffic": None,
    }
    e2e = None
    if not args.no_e2e:
        hl = torch.from_numpy(lhs).pin_memory()
        hr = torch.from_numpy(rhs).pin_memory()
        hz = torch.empty((n, n), dtype=hl.dtype).pin_memory()
        fn = afmm.afmm_case_a if cfg.case == "a" else afmm.afmm_case_b
        devs = dev
        res = fn(hl.numpy(), hr.numpy(), out=hz.numpy(), mode=args.mode, devices=devs, timing=True)
        reps = max(1, min(args.steps, 5))
        t0 = time.perf_counter()
        dev_ms = []
        for _ in range(reps):
            res = fn(hl.numpy(), hr.numpy(), out=hz.numpy(), mode=args.mode, devices=devs,
                     timing=True)
            dev_ms.append(res.timing["total_ms"])
        secs = (time.perf_counter() - t0) / reps
        e2e = {"value": res.counts.additions / secs, "unit": UNIT,
               "h2d_bytes_per_step": 2 * n * n * es, "d2h_bytes_per_step": n * n * es,
               "ms_per_step": secs * 1e3, "device_ms_per_step": statistics.median(dev_ms),
               "steps": reps,
               "api": f"afmm_case_{cfg.case}_{'f32' if es == 4 else 'f64'} (C ABI, host buffers, "
                      f"options.num_devices={G})"}
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": G, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f32" if es == 4 else "f64",
        "data": "synthetic (seeded numpy PCG64, BASELINE.json distributions; no dataset)",
        "config": dict(_config_dict(args, cfg), gather="in-kernel peer stores into GPU 0's Z "
                                                       "(NVLink), no gather step",
                       cuts=[int(c) for c in cuts],
                       **({"test_mode": "AFMM_SINGLE_DEVICE: every shard on cuda:0, not a "
                                        "measurement"} if single else {})),
        "frac_of_fp_add_peak": value / (peak * G),
        "roofline": roofline, "cpu_baseline": None, "e2e": e2e,
        "gpu_launches": launches, "clocks": clocks,
    }
    print(json.dumps(line), flush=True)
    for c in ctxs:
        c.close()


def _secondary(args, afmm, torch, local, peaks):
    """Every other BASELINE configuration at its full size on this GPU: the
    same device-resident step (CUDA events, L2 flushed between steps below
    n = 4096), the repeated-addition kernel's time and its fraction of the
    measured FP-add peak of its dtype. Reported beside the headline so every
    configuration has a driver-run number; not part of `value`."""
    from paper_1308_2400_b200.gen import CONFIGS, make_inputs

    points = [("cfg1", {}), ("cfg2", {})] + [("cfg3", {"d1": d, "mu": m}) for d in (0.1, 0.5, 1.0)
                                              for m in (1, 4, 16)] + [("cfg4", {})]
    points = [(name, kw) for name, kw in points
              if not (name == args.config and (name != "cfg3" or
                                               (kw["d1"], kw["mu"]) == (args.d1, args.mu)))]
    dev = torch.device("cuda", local)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)
    out = {}
    for name, kw in points:
        cfg = CONFIGS[name]
        if cfg.dtype not in peaks:
            peaks[cfg.dtype] = afmm.fp_add_peak(local, cfg.dtype)[0]
        lhs, rhs = make_inputs(name, seed=args.seed, **kw)
        L = torch.from_numpy(lhs).to(dev)
        R = torch.from_numpy(rhs).to(dev)
        Z = torch.empty_like(L)
        ctx = afmm.DeviceContext(local)
        ctx.enable_timing(True)
        steps = 10 if cfg.n <= 4096 else 3
        for _ in range(3):
            ctx.product(cfg.case, L, R, Z)
        ms, kms = [], []
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        for _ in range(steps):
            if cfg.n < 4096:
                flush.fill_(1.0)
            torch.cuda.synchronize()
            e0.record()
            c = ctx.product(cfg.case, L, R, Z)
            e1.record()
            torch.cuda.synchronize()
            ms.append(e0.elapsed_time(e1))
            kms.append(ctx.last_timing()[1])
        form = ctx.last_form()
        ctx.close()
        step = statistics.median(ms)
        k = statistics.median(kms)
        key = name if name != "cfg3" else f"cfg3_d{kw['d1']:g}_mu{kw['mu']}"
        out[key] = {"n": cfg.n, "dtype": "f32" if cfg.dtype == "float32" else "f64",
                    "case": cfg.case, "additions": c.additions, "steps": steps,
                    "ms_per_step": step, "value": c.additions / (step * 1e-3),
                    "frac_of_fp_add_peak": c.additions / (step * 1e-3) / peaks[cfg.dtype],
                    "kernel_ms": k, "kernel_frac": c.additions / (k * 1e-3) / peaks[cfg.dtype],
                    "kernel": form}
        del L, R, Z
    return out


def _reassociated(args, afmm, torch, ctx, cfg, lhs, rhs, L, R, Z, peak):
    """The headline configuration in the two reassociated modes (tolerance
    1e-12 f64 / 1e-5 f32, DESIGN 3.2), device-resident like `value`: reported
    beside the bit-exact headline, never as it. The metric counts the
    additions the product stands for (sum |rep|); "fast-ladder" performs
    fewer, so its performed additions and their pipe fraction are given too."""
    from paper_1308_2400_b200.gen import ladder_additions

    out = {}
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    for mode in ("fast", "fast-ladder"):
        for _ in range(3):
            ctx.product(cfg.case, L, R, Z, mode=mode)
        ms, kms = [], []
        for _ in range(3):
            torch.cuda.synchronize()
            e0.record()
            c = ctx.product(cfg.case, L, R, Z, mode=mode)
            e1.record()
            torch.cuda.synchronize()
            ms.append(e0.elapsed_time(e1))
            kms.append(ctx.last_timing()[1])
        step, k = statistics.median(ms), statistics.median(kms)
        out[mode] = {"ms_per_step": step, "steps": 3, "value": c.additions / (step * 1e-3),
                     "frac_of_fp_add_peak": c.additions / (step * 1e-3) / peak, "kernel_ms": k}
        if mode == "fast-ladder":
            performed = ladder_additions(cfg.case, lhs, rhs)
            out[mode]["performed_additions"] = performed
            out[mode]["performed_frac_of_fp_add_peak"] = performed / (k * 1e-3) / peak
    return out


def _e2e(args, afmm, dist, torch, world, rank, local, cfg, lhs, rhs, es, job_adds, sharded, L,
         R, Z):
    """Same metric with pinned host operands copied in and Z copied out every step."""
    n = lhs.shape[0]
    hl = torch.from_numpy(lhs).pin_memory()
    hr = torch.from_numpy(rhs).pin_memory()
    hz = torch.empty((n, n), dtype=hl.dtype).pin_memory()
    hl_np, hr_np, hz_np = hl.numpy(), hr.numpy(), hz.numpy()
    fn = afmm.afmm_case_a if cfg.case == "a" else afmm.afmm_case_b
    if world > 1:
        from paper_1308_2400_b200.distributed import ShardedProduct

        nccl = os.environ.get("AFMM_DIST_BACKEND", "nccl") == "nccl"
        chunk = (n + world - 1) // world
        c0, c1 = min(n, rank * chunk), min(n, (rank + 1) * chunk)
        Lp = torch.zeros((world * chunk, n), dtype=L.dtype, device=L.device)
        Rp = torch.zeros((world * chunk, n), dtype=R.dtype, device=R.device)
        S = torch.empty((n, n), dtype=L.dtype, device=L.device)
        local = ShardedProduct(sharded.ctx, dist, rank, world, gather="none")

    def step():
        if world == 1:
            # the reference-facing call: afmm_case_{a,b}_{f32,f64}(host ptrs) via the C ABI
            r = fn(hl_np, hr_np, device=local, out=hz_np, mode=args.mode, timing=True)
            dev_ms.append(r.timing["total_ms"])
        else:
            # each rank: H2D of its 1/world row chunk of X and Y, all-gather
            # over NCCL (NVLink), its row slab, D2H of that slab
            if nccl:
                Lp[c0:c1].copy_(hl[c0:c1], non_blocking=True)
                Rp[c0:c1].copy_(hr[c0:c1], non_blocking=True)
                # (whole padded chunks: the last rank's is short when world
                # does not divide n; the padding rows stay zero)
                p0, p1 = rank * chunk, (rank + 1) * chunk
                dist.all_gather_into_tensor(Lp, Lp[p0:p1].clone())
                dist.all_gather_into_tensor(Rp, Rp[p0:p1].clone())
            else:  # gloo (functional test): gather host chunks, then one copy
                for src, dst in ((hl, Lp), (hr, Rp)):
                    parts = [torch.empty_like(torch.zeros(chunk, n, dtype=src.dtype))
                             for _ in range(world)]
                    mine = torch.zeros(chunk, n, dtype=src.dtype)
                    mine[: c1 - c0] = src[c0:c1]
                    dist.all_gather(parts, mine)
                    dst.copy_(torch.cat(parts))
            local.run(cfg.case, Lp[:n], Rp[:n], None, S, mode=args.mode)
            r0, r1 = int(local.cuts[rank]), int(local.cuts[rank + 1])
            hz[r0:r1].copy_(S[: r1 - r0], non_blocking=True)
            torch.cuda.synchronize()

    reps = max(1, min(args.steps, 5))
    dev_ms = []
    for _ in range(1):
        step()
    dev_ms.clear()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        step()
    torch.cuda.synchronize()
    secs = (time.perf_counter() - t0) / reps
    if world > 1:
        on_cpu = os.environ.get("AFMM_DIST_BACKEND", "nccl") != "nccl"
        t = torch.tensor([secs], dtype=torch.float64, device="cpu" if on_cpu else "cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        secs = float(t[0])
    pageable = None
    if world == 1:
        # the same call on PAGEABLE buffers (what a std::vector-backed DenseMatrix
        # or a numpy caller passes): the staged copy pipeline (DESIGN 5)
        out_pg = np.empty_like(lhs)
        fn(lhs, rhs, device=local, out=out_pg, mode=args.mode)
        t1 = time.perf_counter()
        for _ in range(2):
            fn(lhs, rhs, device=local, out=out_pg, mode=args.mode)
        secs_pg = (time.perf_counter() - t1) / 2
        pageable = {"value": job_adds / secs_pg, "unit": UNIT, "ms_per_step": secs_pg * 1e3,
                    "steps": 2}
    return {"value": job_adds / secs, "unit": UNIT, "pageable_host_buffers": pageable,
            "h2d_bytes_per_step": 2 * n * n * es, "d2h_bytes_per_step": n * n * es,
            "ms_per_step": secs * 1e3, "steps": reps,
            "device_ms_per_step": statistics.median(dev_ms) if dev_ms else None,
            "api": "afmm_case_%s_%s (C ABI, host buffers)" % (cfg.case, "f32" if es == 4 else "f64")
            if world == 1 else "per rank: H2D of its 1/N row chunk of X and Y, NCCL all-gather, "
                               "its row slab (cut by predicted time), D2H of the slab"}


def _hbm_check(traffic):
    """The kernel's DRAM bandwidth (ncu bytes per launch / launch time) against the
    driver-measured HBM copy bandwidth: shows the HBM roofline is not the bound."""
    if not traffic:
        return None
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            peak = float(json.load(f)["hbm_gbs"])
        src = "MEASURED_PEAKS.json hbm_gbs"
    except (OSError, ValueError, KeyError):
        peak, src = 7700.0, "B200 nominal (MEASURED_PEAKS.json absent)"
    gbs = traffic["bytes_per_launch"] / traffic["kernel_time_s"] / 1e9
    return {"dram_GBps": gbs, "hbm_peak_GBps": peak, "frac": gbs / peak, "peak_source": src}


def _ncu_traffic(config):
    """dram bytes per launch of k_bform from the committed ncu --set full capture."""
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(path) as f:
            d = json.load(f)
        entry = d.get(config)
        return entry
    except (OSError, ValueError):
        return None


if __name__ == "__main__":
    main()
