#!/usr/bin/env python
"""bench.py -- fused fp16 GEMM + bias + ReLU throughput on B200 (driver contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload NAME] [--impl ours|reference]

A "step" is one pass of the whole hot path over one batch of
synthetic input.  Default workload (BASELINE.json configs[1], the configuration the metric is
quoted on, at its largest size): M = N = K = 8192, bias (row) + ReLU, fp16 out, in all four
operand layouts rr/rc/cr/cc -> 4 fused launches per step.  Each rank runs its own independent
problem (seeded by rank): no collective on the data path, weak scaling.

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
    # name: (batch, M, N, K, layouts, prologue)
    "square8192": (1, 8192, 8192, 8192, ("rr", "rc", "cr", "cc"), None),
    "square4096": (1, 4096, 4096, 4096, ("rr", "rc", "cr", "cc"), None),
    "square2048": (1, 2048, 2048, 2048, ("rr", "rc", "cr", "cc"), None),
    "square1024": (1, 1024, 1024, 1024, ("rr", "rc", "cr", "cc"), None),
    "deepbench_a": (1, 5124, 700, 2048, ("rr", "rc"), None),
    "deepbench_b": (1, 35, 8457, 2560, ("rr", "rc"), None),
    "prologue4096": (1, 4096, 4096, 4096, ("rr",), "scale_k"),
    "batched64x2048": (64, 2048, 2048, 2048, ("rr",), None),
}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--workload", default="square8192", choices=sorted(WORKLOADS))
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


def workload_config(name, world):
    batch, M, N, K, layouts, pro = WORKLOADS[name]
    cfg = {"workload": f"{name}: M=N=K={M}" if M == N == K else f"{name}: M={M} N={N} K={K}",
           "M": M, "N": N, "K": K, "batch_per_gpu": batch, "layouts": list(layouts),
           "epilogue": "bias_relu", "bias": "row (length N)", "prologue": pro or "none", "out": "f16",
           "global_batch": batch * len(layouts) * world,
           "parallelism": f"dp{world} (independent problem per GPU, no collective)"}
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
    batch, M, N, K, layouts, pro = WORKLOADS[args.workload]
    cfg = workload_config(args.workload, 1)
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
def measured_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        mp = json.load(open(p))
        return float(mp["bf16_tflops"]), float(mp.get("bf16_tflops_sustained", 0)) or None, "measured"
    except Exception:
        return 1590.0, 1400.0, "fallback (B200_PROFILING.md)"


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


def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_2006_12645_b200 as ge
    import workloads

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    ge.load_library()
    batch, M, N, K, layouts, pro = WORKLOADS[args.workload]
    cfg = workload_config(args.workload, world)
    seed = 1000 + rank

    # ---- synthetic operands (seeded per rank, generated on the device: timing excludes them)
    g = torch.Generator(device=dev)
    g.manual_seed(seed)
    def U(*shape):
        return (torch.rand(*shape, generator=g, device=dev, dtype=torch.float32) * 2 - 1).half()
    ld8 = lambda n: (n + 7) // 8 * 8           # TMA needs 16-byte row pitch: pad leading dimensions

    def operand(rows, cols, lay):
        """Logical (batch, rows, cols) fp16 operand stored row- ('r') or column-major ('c'), ld padded."""
        if lay == "r":
            return U(batch, rows, ld8(cols))[:, :, :cols]
        return U(batch, cols, ld8(rows))[:, :, :rows].transpose(1, 2)

    # Operand sets are rotated between steps so the working set exceeds the 126 MB L2 (no flush
    # kernel inside the timed region); one set when a single step already streams > 3x L2.
    set_bytes = sum(2 * (M * ld8(K) + K * ld8(N)) * batch for _ in layouts)
    n_sets = max(1, min(64, -(-int(3 * 126e6) // set_bytes)))
    sets = [[(lay, operand(M, K, lay[0]), operand(K, N, lay[1])) for lay in layouts] for _ in range(n_sets)]
    ops = sets[0]
    bias = U(N)
    scale = (torch.rand(K, generator=g, device=dev) + 0.5) if pro == "scale_k" else None
    C = torch.empty(batch, M, ld8(N), dtype=torch.float16, device=dev)[:, :, :N]
    cfg["l2"] = (f"{n_sets} operand sets rotated across steps ({n_sets * set_bytes / 1e6:.0f} MB working set > "
                 f"126 MB L2), no flush")
    if ld8(N) != N or ld8(K) != K or ld8(M) != M:
        cfg["padding"] = "leading dimensions padded to a multiple of 8 elements (16-byte TMA pitch)"
    stream = torch.cuda.current_stream()

    def launch(lay, A, B):
        if batch == 1:
            ge.gemm_epilogue(A[0], B[0], bias, prologue=pro, scale=scale, out=C[0])
        else:
            ge.gemm_epilogue_batched(A, B, bias, prologue=pro, scale=scale, out=C)

    step_no = [0]

    def step_eager():
        cur = sets[step_no[0] % n_sets]
        step_no[0] += 1
        for lay, A, B in cur:
            launch(lay, A, B)

    for _ in range(args.warmup):
        step_eager()
    torch.cuda.synchronize()

    # A step is replayed from a CUDA graph captured per operand set (the 4 launches are plain
    # cudaLaunchKernelEx calls on the capturing stream): no host launch overhead in the timed region.
    graphs = None
    launches_per_step = len(layouts)
    if not args.no_graph:
        graphs = []
        for cur in sets:
            gr = torch.cuda.CUDAGraph()
            with torch.cuda.graph(gr):
                for lay, A, B in cur:
                    launch(lay, A, B)
            graphs.append(gr)
        for i in range(max(1, args.warmup)):
            graphs[i % n_sets].replay()
        torch.cuda.synchronize()

    # ---- timed region
    step_ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
               for _ in range(args.steps)]
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    n_launch0 = ge.launch_count()
    with ClockSampler(local) as clk:
        t0.record(stream)
        for s in range(args.steps):
            step_ev[s][0].record(stream)
            if graphs is not None:
                graphs[s % n_sets].replay()
            else:
                step_eager()
            step_ev[s][1].record(stream)
        t1.record(stream)
        torch.cuda.synchronize()
    n_launches = (ge.launch_count() - n_launch0) if graphs is None else launches_per_step * args.steps
    if world > 1:
        dist.barrier()
    ms = t0.elapsed_time(t1)
    # the step holds only our kernels, back to back: per-launch time = step time / launches
    kern_ms = [a.elapsed_time(b) / launches_per_step for (a, b) in step_ev]
    kern_avg_ms = sum(kern_ms) / len(kern_ms)
    if world > 1:
        tt = torch.tensor([ms], device=dev, dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms = float(tt.item())
    flop_per_launch = 2.0 * M * N * K * batch
    flop_total = flop_per_launch * len(ops) * args.steps * world
    value = flop_total / (ms * 1e-3) / 1e12

    # ---- end to end through the host-buffer C-ABI entry point
    e2e = None
    if args.e2e_steps > 0:
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
        hA = [host_copy(A, lay[0]) for lay, A, B in ops]
        hB = [host_copy(B, lay[1]) for lay, A, B in ops]
        Ah, Bh = [x for x, _ in hA], [x for x, _ in hB]
        bh = bias.cpu().pin_memory()
        sh = scale.cpu().pin_memory() if scale is not None else None
        Ch = torch.empty(batch, M, ld8(N), dtype=torch.float16).pin_memory()[:, :, :N]

        def e2e_step():
            for i in range(len(ops)):
                ge.gemm_epilogue_host(Ah[i], Bh[i], bh, prologue=pro, scale=sh, out=Ch)
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
        h2d = sum(na + nb + bh.numel() * 2 + (sh.numel() * 4 if sh is not None else 0)
                  for (_, na), (_, nb) in zip(hA, hB))
        d2h = len(ops) * batch * M * N * 2
        e2e = {"value": flop_per_launch * len(ops) * args.e2e_steps * world / (ems * 1e-3) / 1e12, "unit": UNIT,
               "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h, "steps": args.e2e_steps,
               "path": "gemm_epilogue_host (C ABI, pinned host buffers)"}
        ge.load_library().ge_release_workspace()

    clocks = clk.summary()
    if world > 1:
        allc = [None] * world
        dist.all_gather_object(allc, clocks)
        clocks = dict(allc[0])
        clocks["per_rank_sm_mhz"] = [c.get("sm_mhz") for c in allc]
        clocks["reasons"] = sorted({r for c in allc for r in c.get("reasons", [])})

    if rank == 0:
        peak, peak_sus, peak_src = measured_peak()
        achieved = flop_per_launch / (kern_avg_ms * 1e-3) / 1e12
        traffic, tsrc = ncu_traffic(args.workload)
        roofline = {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                    "frac": achieved / peak, "traffic": traffic,
                    "peak_source": f"{peak_src} bf16 burst (MEASURED_PEAKS.json bf16_tflops; fp16 = bf16 nominal)",
                    "frac_of_sustained": (achieved / peak_sus) if peak_sus else None,
                    "frac_of_spec_2250": achieved / 2250.0,
                    "kernel": "ge_fused_kernel (one launch per GEMM)",
                    "kernel_avg_ms": kern_avg_ms,
                    "launch_mode": "CUDA graph replay per step" if graphs is not None else "eager",
                    "traffic_source": tsrc}
        comparators = None
        if not args.no_comparators and batch == 1:
            comparators = compare_torch(torch, sets, bias, M, N, K, stream, iters=args.steps * len(layouts))
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": "f16", "accumulate": "f32",
                "data": "synthetic (seeded U(-1,1) fp16)", "config": cfg,
                "roofline": roofline, "e2e": e2e, "gpu_launches": n_launches, "clocks": clocks,
                "comparators": comparators}
        if not args.no_cpu_baseline:
            rate, cores, desc, _ = oracle_rate(M, N, K, seed=7, budget_s=12.0)
            line["cpu_baseline"] = {"value": rate, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": desc}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def compare_torch(torch, sets, bias, M, N, K, stream, iters=10):
    """Library reference points on the same box and the same rotating operand sets (not the product):
    torch unfused matmul + add + relu (cuBLAS + 2 elementwise kernels, the paper's baseline shape,
    PAPER.md:1255-1260), torch._addmm_activation (cuBLASLt bias+ReLU epilogue) and plain
    torch.matmul.  Each is replayed from CUDA graphs like our step; first layout of each set."""
    out = {}
    fl = 2.0 * M * N * K

    def t(fn, it=iters):
        graphs = []
        for cur in sets:
            lay, A, B = cur[0]
            a, b = A[0], B[0]
            fn(a, b)
            gr = torch.cuda.CUDAGraph()
            with torch.cuda.graph(gr):
                fn(a, b)
            graphs.append(gr)
        for i in range(3):
            graphs[i % len(graphs)].replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for i in range(it):
            graphs[i % len(graphs)].replay()
        e1.record(stream)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / it * 1e-3
    try:
        out["torch_unfused_matmul_add_relu"] = fl / t(lambda a, b: torch.relu_(torch.matmul(a, b).add_(bias))) / 1e12
        out["torch_matmul_only"] = fl / t(lambda a, b: torch.matmul(a, b)) / 1e12
        out["cublaslt_addmm_relu"] = fl / t(lambda a, b: torch._addmm_activation(bias, a, b)) / 1e12
        out["layout"] = sets[0][0][0]
        out["protocol"] = (f"CUDA graph replay, same rotating operand sets, {iters} launches each "
                           "(as many as our timed region)")
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
