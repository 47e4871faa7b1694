#!/usr/bin/env python
"""bench.py -- fused fp16 GEMM + bias + ReLU throughput on B200 (driver contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload NAME] [--impl ours|reference]

A "step" is one pass of the whole hot path over one batch of
synthetic input.  Default workload at N = 1 (BASELINE.json configs[1], the configuration the
metric is quoted on, at its largest size): M = N = K = 8192, bias (row) + ReLU, fp16 out, in all
four operand layouts rr/rc/cr/cc -> 4 fused launches per step.  Default at N > 1 (north_star:
"scaling ... to 8 GPUs on sharded batches", BASELINE.json configs[4]): batched64x2048, a GLOBAL
batch of 64 items of 2048^3 sharded by batch with sharded.sharded_gemm_epilogue_batched (rank r
owns items [r*64/N, (r+1)*64/N), generated from per-item seeds so shards do not depend on N), no
collective on the data path, strong scaling; the N = 1 line carries that workload's N = 1 point
as "scale_series" so the series is comparable.

Timing: W untimed warm-up steps; K timed steps bracketed by barrier + synchronize, CUDA events
on the launching stream, max over ranks.  Operands (256 MiB per layout per step) exceed the
126 MB L2, so no flush is needed.  NVML samples SM clocks / throttle reasons during the timed
region.  `e2e` repeats the step through the host-buffer C-ABI entry (gemm_epilogue_host):
pinned host inputs copied in and C copied out inside the timed region.

`--impl reference` times the CPU oracle (oracle/, the arm the driver divides by) on a bounded
sample of the same workload; only rank 0 works under torchrun.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "TFLOP/s fused GEMM+bias+ReLU (fp16 in, fp32 acc) and % of B200 tensor peak"
UNIT = "TFLOP/s"

WORKLOADS = {
    # name: (batch, M, N, K, layouts, prologue); batched64x2048's batch is GLOBAL (sharded over ranks)
    "square256": (1, 256, 256, 256, ("rr",), None),
    "square8192": (1, 8192, 8192, 8192, ("rr", "rc", "cr", "cc"), None),
    "square4096": (1, 4096, 4096, 4096, ("rr", "rc", "cr", "cc"), None),
    "square2048": (1, 2048, 2048, 2048, ("rr", "rc", "cr", "cc"), None),
    "square1024": (1, 1024, 1024, 1024, ("rr", "rc", "cr", "cc"), None),
    "deepbench_a": (1, 5124, 700, 2048, ("rr", "rc"), None),
    "deepbench_b": (1, 35, 8457, 2560, ("rr", "rc"), None),
    "prologue4096": (1, 4096, 4096, 4096, ("rr",), "scale_k"),
    "hadamard4096": (1, 4096, 4096, 4096, ("rr",), "hadamard"),
    "batched64x2048": (64, 2048, 2048, 2048, ("rr",), None),
}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--workload", default="auto", choices=["auto"] + sorted(WORKLOADS),
                    help="auto: square8192 at N = 1, batched64x2048 (global batch sharded) at N > 1")
    ap.add_argument("--gather", action="store_true", help="batched64x2048 at N > 1: also time the optional "
                    "NCCL all-gather of the output shards (reported separately, off the hot path)")
    ap.add_argument("--no-scale-series", action="store_true")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-comparators", action="store_true")
    ap.add_argument("--no-graph", action="store_true", help="launch from Python every step instead of replaying "
                    "a captured CUDA graph per operand set")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


SHARDED = ("batched64x2048",)       # global batch sharded over ranks (strong scaling)


def resolve_workload(name, world):
    if name == "auto":
        return "square8192" if world == 1 else "batched64x2048"
    return name


def workload_config(name, world, rank=0):
    batch, M, N, K, layouts, pro = WORKLOADS[name]
    cfg = {"workload": f"{name}: M=N=K={M}" if M == N == K else f"{name}: M={M} N={N} K={K}",
           "M": M, "N": N, "K": K, "batch_per_gpu": batch, "layouts": list(layouts),
           "epilogue": "bias_relu", "bias": "row (length N)", "prologue": pro or "none", "out": "f16",
           "global_batch": batch * len(layouts) * world,
           "parallelism": f"dp{world} (independent problem per GPU, no collective)"}
    if name in SHARDED:
        from paper_2006_12645_b200 import sharded
        lo, hi = sharded.shard_range(batch, rank, world)
        cfg.update({"batch_per_gpu": hi - lo, "global_batch": batch,
                    "bias": "row, one per item (length N)",
                    "parallelism": f"dp{world}: global batch {batch} sharded by batch (sharded_gemm_epilogue_batched, "
                                   f"rank r owns items [r*{batch}/{world}, (r+1)*{batch}/{world})), no collective"})
    return cfg


# ------------------------------------------------------------------ clocks (NVML)
class ClockSampler:
    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
               0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
               0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}

    def __init__(self, device_index):
        self.samples, self.reasons, self.stop = [], 0, threading.Event()
        self.ok = False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception as e:  # pragma: no cover - no NVML
            self.err = str(e)

    def _run(self):
        while not self.stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                self.reasons |= self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
            except Exception:
                pass
            time.sleep(0.01)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self.stop.set()
            self.t.join()

    def summary(self):
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvml unavailable"]}
        s = sorted(self.samples)
        names = [n for b, n in self.REASONS.items() if self.reasons & b and n != "gpu_idle"]
        return {"sm_mhz": s[len(s) // 2], "sm_max_mhz": self.max_mhz, "reasons": names, "samples": len(s)}


# ------------------------------------------------------------------ CPU oracle (reference arm / baseline)
def oracle_rate(M, N, K, seed, budget_s, min_side=8, max_side=1024):
    """Time the CPU oracle (as it stands) on square output blocks of the rr problem; returns
    (TFLOP/s, cores, sample description).  The block side is calibrated to ~budget_s."""
    import numpy as np
    import oracle
    import workloads
    cores = oracle.default_threads()
    g = np.random.default_rng(seed)
    # build only the rows/cols the sample touches (operands are generated in full for simplicity
    # only when they are small; for the big shapes we draw the sampled slices directly)
    def block(side):
        rows = np.sort(g.choice(M, size=min(side, M), replace=False))
        cols = np.sort(g.choice(N, size=min(side, N), replace=False))
        A = workloads.uniform_f16((len(rows), K), seed * 7 + 1)       # the sampled rows of A
        B = workloads.uniform_f16((K, len(cols)), seed * 7 + 2)       # the sampled columns of B
        bias = workloads.uniform_f16((len(cols),), seed * 7 + 3)
        t0 = time.perf_counter()
        oracle.gemm_epilogue(A, B, len(rows), len(cols), K, layoutA="row", layoutB="row", bias=bias,
                             bias_mode="row", nthreads=cores)
        return time.perf_counter() - t0, len(rows) * len(cols)
    t, n = block(min(64, M, N))
    per_el = t / n
    side = int(max(min_side, min(max_side, (budget_s / per_el) ** 0.5)))
    t, n = block(side)
    rate = 2.0 * n * K / t / 1e12
    desc = (f"{min(side, M)}x{min(side, N)} output block (random rows/cols) of the M={M} N={N} K={K} rr problem, "
            f"full K, fp64 oracle on {cores} host threads, {t:.1f} s")
    return rate, cores, desc, t


def run_reference(args):
    rank, world, local = dist_env()
    if rank != 0:
        return 0
    name = resolve_workload(args.workload, world)
    batch, M, N, K, layouts, pro = WORKLOADS[name]
    cfg = workload_config(name, world, 0)
    # each step: one bounded sample, sized so warmup+steps fit in ~120 s
    per_step = max(0.05, 120.0 / max(1, args.steps + args.warmup))
    rate, cores, desc, t = oracle_rate(M, N, K, seed=0, budget_s=per_step)
    times = []
    side = None
    import oracle  # noqa: F401
    for i in range(args.warmup + args.steps):
        r, _, d, tt = oracle_rate(M, N, K, seed=i + 1, budget_s=per_step)
        if i >= args.warmup:
            times.append((r, tt))
            desc = d
    vals = [r for r, _ in times]
    value = sorted(vals)[len(vals) // 2] if vals else rate
    ms = 1e3 * sum(tt for _, tt in times) / max(1, len(times))
    line = {"metric": METRIC, "value": value, "unit": UNIT, "impl": "reference", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic", "config": cfg,
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle",
                             "sample": "per step: " + desc},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------ our arm
def measured_peaks():
    """(bf16 burst TF/s, sustained TF/s, HBM GB/s, source) from the driver-written MEASURED_PEAKS.json,
    else the B200_PROFILING.md fallbacks."""
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        mp = json.load(open(p))
        return (float(mp["bf16_tflops"]), float(mp.get("bf16_tflops_sustained", 0)) or None, float(mp["hbm_gbs"]),
                "measured")
    except Exception:
        return 1590.0, 1400.0, 6500.0, "fallback (B200_PROFILING.md)"


def ncu_traffic(workload):
    """Per-launch DRAM bytes (read + write) of the fused kernel from the committed ncu --set full
    summary (profiles/), or None."""
    p = os.path.join(ROOT, "profiles", "ncu_summary.json")
    try:
        d = json.load(open(p))
        e = d["kernels"][workload]
        return float(e["dram_bytes_read"]) + float(e["dram_bytes_write"]), e.get("source")
    except Exception:
        return None, None


def algorithmic_bytes(batch, M, N, K, pro):
    """What one launch must move: A, B, C (fp16) per item, the ROW bias per item
    (bench uses one per item for batches, one shared otherwise) and the SCALE_K vector."""
    per_item = 2 * M * K + 2 * K * N + 2 * M * N
    bias = 2 * N * (batch if batch > 1 else 1)
    return batch * per_item + bias + (4 * K if pro == "scale_k" else 0) + (2 * M * K if pro == "hadamard" else 0)


class Workload:
    """Synthetic operands of one bench workload on this rank, the fused launch of one step, and
    CUDA graphs of the step.  Operand sets rotate between steps so the working set exceeds the
    126 MB L2 (no flush kernel in the timed region)."""

    def __init__(self, name, dev, rank, world, torch, ge):
        self.name, self.torch, self.ge = name, torch, ge
        gbatch, M, N, K, layouts, pro = WORKLOADS[name]
        self.M, self.N, self.K, self.layouts, self.pro = M, N, K, layouts, pro
        self.sharded = name in SHARDED
        if self.sharded:
            from paper_2006_12645_b200 import sharded
            self.lo, self.hi = sharded.shard_range(gbatch, rank, world)
            self.batch, self.gbatch = self.hi - self.lo, gbatch
        else:
            self.lo, self.hi, self.batch, self.gbatch = 0, gbatch, gbatch, gbatch * world
        ld8 = self.ld8 = lambda n: (n + 7) // 8 * 8           # TMA needs a 16-byte row pitch: pad ld
        batch = self.batch
        g = torch.Generator(device=dev)

        def U(*shape, seed=None):
            if seed is not None:
                g.manual_seed(seed)
            return (torch.rand(*shape, generator=g, device=dev, dtype=torch.float32) * 2 - 1).half()

        def operand(rows, cols, lay, which, rot):
            """Logical (batch, rows, cols) fp16 operand stored row- ('r') or column-major ('c'), ld padded.
            Sharded batches draw item b from its own seed, so a rank's items do not depend on N."""
            shape = (rows, ld8(cols)) if lay == "r" else (cols, ld8(rows))
            if self.sharded:
                x = torch.stack([U(*shape, seed=(4 << 24) + (rot << 16) + (b << 2) + which)
                                 for b in range(self.lo, self.hi)]) if batch else \
                    torch.empty((0,) + shape, dtype=torch.float16, device=dev)
            else:
                x = U(batch, *shape, seed=1000 + rank + 7919 * (rot * 4 + which))
            return x[:, :, :cols] if lay == "r" else x[:, :, :rows].transpose(1, 2)

        set_bytes = max(1, sum(2 * (M * ld8(K) + K * ld8(N)) * batch for _ in layouts))
        self.n_sets = max(1, min(64, -(-int(3 * 126e6) // set_bytes)))
        self.sets = [[(lay, operand(M, K, lay[0], 1, r), operand(K, N, lay[1], 2, r)) for lay in layouts]
                     for r in range(self.n_sets)]
        self.set_bytes = set_bytes
        if self.sharded:
            self.bias = torch.stack([U(N, seed=(4 << 24) + (b << 2) + 3) for b in range(self.lo, self.hi)]) \
                if batch else torch.empty((0, N), dtype=torch.float16, device=dev)
        else:
            self.bias = U(N, seed=1000 + rank + 31)
        self.scale = (torch.rand(K, generator=g, device=dev) + 0.5) if pro == "scale_k" else None
        if pro == "hadamard":          # the M x K tile S, stored in A's layout, U(0.5, 1.5)
            lay = layouts[0][0]
            S = (torch.rand((M, ld8(K)) if lay == "r" else (K, ld8(M)), generator=g, device=dev) + 0.5).half()
            self.scale = S[:, :K] if lay == "r" else S[:, :M].t()
        self.C = torch.empty(max(batch, 1), M, ld8(N), dtype=torch.float16, device=dev)[:batch, :, :N]
        self.step_no = 0

    def launch(self, A, B):
        ge = self.ge
        if self.sharded:
            from paper_2006_12645_b200 import sharded
            sharded.sharded_gemm_epilogue_batched(A, B, self.bias, presliced=True, total_batch=self.gbatch,
                                                  prologue=self.pro, scale=self.scale, out=self.C)
        elif self.batch == 1:
            ge.gemm_epilogue(A[0], B[0], self.bias, prologue=self.pro, scale=self.scale, out=self.C[0])
        else:
            ge.gemm_epilogue_batched(A, B, self.bias, prologue=self.pro, scale=self.scale, out=self.C)

    def launches_per_step(self):
        return len(self.layouts) if self.batch > 0 else 0

    def step_eager(self):
        cur = self.sets[self.step_no % self.n_sets]
        self.step_no += 1
        for lay, A, B in cur:
            self.launch(A, B)

    def capture(self, steps, first=0):
        """One CUDA graph holding `steps` consecutive steps (operand sets rotating as in eager
        steps): the launches replay back to back with no host work or graph-launch gap between
        steps (the task's "capture launch-bound inner loops in CUDA graphs")."""
        torch = self.torch
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gr):
            for i in range(steps):
                for lay, A, B in self.sets[(first + i) % self.n_sets]:
                    self.launch(A, B)
        return gr

    def flop_per_launch(self):
        return 2.0 * self.M * self.N * self.K * self.batch


def time_steps(w, steps, warmup, stream, torch, dist, world, graph=True, clock=None):
    """W eager warm-up steps; then (graph mode) the K timed steps captured into ONE CUDA graph and a
    W-step warm-up graph replayed first; the timed region (barrier + synchronize on both sides, CUDA
    events on the launching stream) replays the K-step graph once (or, eager, runs K steps from
    Python).  Returns (ms total (max over ranks), per-launch kernel ms on this rank, #launches)."""
    for _ in range(warmup):
        w.step_eager()
    torch.cuda.synchronize()
    g_timed = None
    if graph:
        g_warm = w.capture(max(1, warmup), first=0)
        g_timed = w.capture(steps, first=0)
        g_warm.replay()
        torch.cuda.synchronize()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    n0 = w.ge.launch_count()
    ctx = clock if clock is not None else _NullCtx()
    with ctx:
        gpu_busy(torch, stream)
        t0.record(stream)
        if g_timed is not None:
            g_timed.replay()
        else:
            for _ in range(steps):
                w.step_eager()
        t1.record(stream)
        torch.cuda.synchronize()
    n_launch = (w.ge.launch_count() - n0) if g_timed is None else w.launches_per_step() * steps
    if world > 1:
        dist.barrier()
    ms = t0.elapsed_time(t1)
    kern_ms = ms / max(1, steps * w.launches_per_step())    # only our kernels run in the region
    if world > 1:
        tt = torch.tensor([ms], device=w.C.device, dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms = float(tt.item())
    return ms, kern_ms, n_launch


def gpu_busy(torch, stream):
    """Queue ~1 ms of device spin ahead of the start event: the host-side submission of the timed
    graph (or of the first eager launches) then overlaps it, so the CUDA-event region holds only the
    kernels being timed back to back, not the host's launch latency.  The spin runs before t0."""
    with torch.cuda.stream(stream):
        torch.cuda._sleep(2_000_000)


class _NullCtx:
    def __enter__(self):
        return self

    def __exit__(self, *a):
        return False


def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_2006_12645_b200 as ge

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    ge.load_library()
    name = resolve_workload(args.workload, world)
    w = Workload(name, dev, rank, world, torch, ge)
    cfg = workload_config(name, world, rank)
    M, N, K, pro = w.M, w.N, w.K, w.pro
    cfg["l2"] = (f"{w.n_sets} operand sets rotated across steps ({w.n_sets * w.set_bytes / 1e6:.0f} MB working set > "
                 f"126 MB L2), no flush")
    if w.ld8(N) != N or w.ld8(K) != K or w.ld8(M) != M:
        cfg["padding"] = "leading dimensions padded to a multiple of 8 elements (16-byte TMA pitch)"
    stream = torch.cuda.current_stream()

    clk = ClockSampler(local)
    ms, kern_avg_ms, n_launches = time_steps(w, args.steps, args.warmup, stream, torch, dist, world,
                                             graph=not args.no_graph, clock=clk)
    flop_step_global = 2.0 * M * N * K * len(w.layouts) * w.gbatch
    value = flop_step_global * args.steps / (ms * 1e-3) / 1e12

    # ---- optional all-gather of the output shards (off the hot path; algbw / busbw, nccl-tests convention)
    gather = None
    if args.gather and w.sharded and world > 1:
        from paper_2006_12645_b200 import sharded
        sharded.gather_rows(w.C, w.gbatch)
        torch.cuda.synchronize()
        dist.barrier()
        g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        g0.record(stream)
        reps = 5
        for _ in range(reps):
            sharded.gather_rows(w.C, w.gbatch)
        g1.record(stream)
        torch.cuda.synchronize()
        gms = g0.elapsed_time(g1) / reps
        tt = torch.tensor([gms], device=dev, dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        gms = float(tt.item())
        nbytes = w.gbatch * M * N * 2
        gather = {"bytes": nbytes, "ms": gms, "algbw_gbs": nbytes / (gms * 1e-3) / 1e9,
                  "busbw_gbs": nbytes / (gms * 1e-3) / 1e9 * (world - 1) / world,
                  "note": "torch.distributed all_gather_into_tensor (NCCL) of the C shards, timed after the steps"}

    # ---- end to end through the host-buffer C-ABI entry point (this rank's items)
    e2e = None
    if args.e2e_steps > 0 and w.batch > 0:
        e2e = run_e2e(args, w, torch, dist, world, stream, dev)
        cfg_e2e_flop = 2.0 * M * N * K * len(w.layouts) * w.gbatch
        e2e["value"] = cfg_e2e_flop * args.e2e_steps / (e2e.pop("ms") * 1e-3) / 1e12

    clocks = clk.summary()
    if world > 1:
        allc = [None] * world
        dist.all_gather_object(allc, clocks)
        clocks = dict(allc[0])
        clocks["per_rank_sm_mhz"] = [c.get("sm_mhz") for c in allc]
        clocks["reasons"] = sorted({r for c in allc for r in c.get("reasons", [])})

    # ---- N = 1 point of the N > 1 default (scale series), measured in the same run
    scale_series = None
    if world == 1 and args.workload == "auto" and not args.no_scale_series:
        ws = Workload("batched64x2048", dev, 0, 1, torch, ge)
        sms_, skm_, _ = time_steps(ws, min(args.steps, 10), 3, stream, torch, dist, 1, graph=not args.no_graph)
        fl = 2.0 * ws.M * ws.N * ws.K * ws.gbatch * min(args.steps, 10)
        scale_series = {"workload": "batched64x2048 (global batch 64 sharded by batch; the default at N > 1)",
                        "value_n1": fl / (sms_ * 1e-3) / 1e12, "unit": UNIT,
                        "kernel_avg_ms": skm_, "steps": min(args.steps, 10)}
        del ws

    if rank == 0:
        peak, peak_sus, hbm, peak_src = measured_peaks()
        flop_launch = w.flop_per_launch()
        bytes_launch = algorithmic_bytes(w.batch, M, N, K, pro)
        ai = flop_launch / max(1.0, bytes_launch)
        ridge = peak * 1e12 / (hbm * 1e9)
        traffic, tsrc = ncu_traffic(name)
        common = {"kernel": "ge_fused_kernel (one launch per GEMM / batch)", "kernel_avg_ms": kern_avg_ms,
                  "launch_mode": ("one CUDA graph replay of the K timed steps (launches back to back)"
                                  if not args.no_graph else "eager"),
                  "traffic": traffic, "traffic_source": tsrc,
                  "algorithmic_flop_per_launch": flop_launch, "algorithmic_bytes_per_launch": bytes_launch,
                  "arithmetic_intensity": ai, "ridge_flop_per_byte": ridge}
        if ai < ridge:
            # HBM-bound shape: GB/s of algorithmic bytes against the measured copy bandwidth
            achieved = bytes_launch / (kern_avg_ms * 1e-3) / 1e9
            roofline = {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s", "frac": achieved / hbm,
                        "peak_source": f"{peak_src} HBM copy bandwidth (MEASURED_PEAKS.json hbm_gbs)",
                        "tflops": flop_launch / (kern_avg_ms * 1e-3) / 1e12, **common}
        else:
            achieved = flop_launch / (kern_avg_ms * 1e-3) / 1e12
            roofline = {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                        "frac": achieved / peak,
                        "peak_source": f"{peak_src} bf16 burst (MEASURED_PEAKS.json bf16_tflops; fp16 = bf16 nominal)",
                        "frac_of_sustained": (achieved / peak_sus) if peak_sus else None,
                        "frac_of_spec_2250": achieved / 2250.0, **common}
        comparators = None
        if not args.no_comparators and w.batch == 1:
            comparators = compare_torch(torch, w, stream, iters=args.steps * len(w.layouts))
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
                "scaling": "strong" if w.sharded else "weak", "vs_baseline": None, "dtype": "f16",
                "accumulate": "f32", "data": "synthetic (seeded U(-1,1) fp16)", "config": cfg,
                "roofline": roofline, "e2e": e2e, "gpu_launches": n_launches, "clocks": clocks,
                "comparators": comparators}
        if gather:
            line["gather"] = gather
        if scale_series:
            line["scale_series"] = scale_series
        if not args.no_cpu_baseline:
            rate, cores, desc, _ = oracle_rate(M, N, K, seed=7, budget_s=36.0, max_side=4096)
            line["cpu_baseline"] = {"value": rate, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": desc}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def run_e2e(args, w, torch, dist, world, stream, dev):
    """The same step through the host-buffer C-ABI entry (gemm_epilogue_host): pinned host inputs
    copied in and C copied out inside the timed region; this rank's items."""
    ge, ld8, batch = w.ge, w.ld8, w.batch

    def host_copy(x, lay):
        """Pinned host copy of a logical (batch, rows, cols) operand, same layout and padded ld."""
        rows, cols = x.shape[1], x.shape[2]
        if lay == "r":
            st_ = torch.empty(batch, rows, ld8(cols), dtype=torch.float16).pin_memory()
            st_[:, :, :cols] = x.cpu()
            return st_[:, :, :cols], st_.numel() * 2
        st_ = torch.empty(batch, cols, ld8(rows), dtype=torch.float16).pin_memory()
        st_[:, :, :rows] = x.transpose(1, 2).cpu()
        return st_[:, :, :rows].transpose(1, 2), st_.numel() * 2
    ops = w.sets[0]
    hA = [host_copy(A, lay[0]) for lay, A, B in ops]
    hB = [host_copy(B, lay[1]) for lay, A, B in ops]
    Ah, Bh = [x for x, _ in hA], [x for x, _ in hB]
    bh = w.bias.cpu().pin_memory()
    sh = w.scale.cpu().pin_memory() if w.scale is not None else None
    Ch = torch.empty(batch, w.M, ld8(w.N), dtype=torch.float16).pin_memory()[:, :, :w.N]

    def e2e_step():
        for i in range(len(ops)):
            if batch == 1:
                ge.gemm_epilogue_host(Ah[i][0], Bh[i][0], bh, prologue=w.pro, scale=sh, out=Ch[0])
            else:
                ge.gemm_epilogue_host(Ah[i], Bh[i], bh, prologue=w.pro, scale=sh, out=Ch)
    e2e_step()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.e2e_steps):
        e2e_step()
    e1.record(stream)
    torch.cuda.synchronize()
    ems = e0.elapsed_time(e1)
    if world > 1:
        tt = torch.tensor([ems], device=dev, dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ems = float(tt.item())
    h2d = sum(na + nb + bh.numel() * 2 + (sh.numel() * 4 if sh is not None else 0) for (_, na), (_, nb) in zip(hA, hB))
    d2h = len(ops) * batch * w.M * w.N * 2
    ge.load_library().ge_release_workspace()
    return {"ms": ems, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
            "steps": args.e2e_steps, "path": "gemm_epilogue_host (C ABI, pinned host buffers)"}


def compare_torch(torch, w, stream, iters=10):
    """Library reference points on the same box and the same rotating operand sets (not the product):
    torch unfused matmul + add + relu (cuBLAS + 2 elementwise kernels, the paper's baseline shape,
    PAPER.md:1255-1260), torch._addmm_activation (cuBLASLt bias+ReLU epilogue) and plain
    torch.matmul.  Each runs as one CUDA graph of the same number of calls as our timed region, over
    the same rotating operand sets and the same layouts in the same order (cuBLAS picks its kernel
    per layout, so both sides switch kernels alike).
    Like-for-like alignment: when N is not a multiple of 8, the library computes the padded
    N' = ld8(N) columns (row-major B: the same padded storage we read; column-major B: a padded
    copy), so its C rows are 16-byte aligned like ours (TFLOP/s still counts the logical 2MNK)."""
    out = {}
    M, N, K = w.M, w.N, w.K
    fl = 2.0 * M * N * K
    Np = w.ld8(N)
    layouts = [lay for lay, _, _ in w.sets[0]]
    pad = Np != N
    bias = w.bias if not pad else torch.cat([w.bias, torch.zeros(Np - N, dtype=w.bias.dtype, device=w.bias.device)])

    def operands(lay, A, B):
        a, b = A[0], B[0]
        if pad and lay[1] == "r":
            b = torch.as_strided(b, (K, Np), (b.stride(0), 1))     # the padded storage row pitch (ld8(N))
        elif pad:
            # col-major B: a copy with Np columns (made here, outside the timed region) so the
            # library's C rows are 16-byte aligned like ours
            bp = torch.zeros((Np, b.stride(1)), dtype=b.dtype, device=b.device)
            bp[:N] = torch.as_strided(b, (N, b.stride(1)), (b.stride(1), 1))
            b = bp[:, :K].t()
        return a, b

    def t(fn, it=iters):
        """One CUDA graph of `it` calls rotating the operand sets, replayed once (our protocol)."""
        # every layout of every operand set, in the order of our steps (the same kernel mix)
        ops = [operands(lay, A, B) for cur in w.sets for lay, A, B in cur]
        for a, b in ops[:2]:
            fn(a, b)
        torch.cuda.synchronize()
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gr):
            for i in range(it):
                fn(*ops[i % len(ops)])
        gr.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        gpu_busy(torch, stream)
        e0.record(stream)
        gr.replay()
        e1.record(stream)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / it * 1e-3
    try:
        bias_for = lambda b: bias if b.shape[1] == bias.shape[0] else w.bias
        out["torch_unfused_matmul_add_relu"] = fl / t(lambda a, b: torch.relu_(torch.matmul(a, b).add_(bias_for(b)))) / 1e12
        out["torch_matmul_only"] = fl / t(lambda a, b: torch.matmul(a, b)) / 1e12
        out["cublaslt_addmm_relu"] = fl / t(lambda a, b: torch._addmm_activation(bias_for(b), a, b)) / 1e12
        out["layouts"] = layouts
        out["ldc"] = Np if pad else N
        out["protocol"] = (f"one CUDA graph of {iters} calls over the same rotating operand sets, replayed once "
                           "(as our timed region)" + ("; N padded to ld8(N) for 16-B aligned C rows" if pad else ""))
    except Exception as e:  # pragma: no cover
        out["error"] = str(e)
    return out


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
