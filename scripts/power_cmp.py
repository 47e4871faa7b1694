"""Dev: sustained TF/s, SM clock and board power of our kernel configs vs cuBLAS(Lt) at one shape.
Each candidate runs graph-replayed for ~SECS seconds with rotating operand sets while a thread
samples NVML; reports TF/s, median SM MHz, median W, and flop/clk/SM (clock-normalised
efficiency: 8192 = the tensor pipe's dense fp16 rate).
usage: power_cmp.py M N K [secs] [cfg ...]   cfg = auto | cublas | lt | BNxCG[m]"""
import sys, os, time, threading, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import pynvml
import paper_2006_12645_b200 as ge

M, N, K = (int(x) for x in sys.argv[1:4])
secs = float(sys.argv[4]) if len(sys.argv) > 4 else 2.0
cfgs = sys.argv[5:] or ["auto", "512x2", "256x2", "lt", "cublas"]
pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(torch.cuda.current_device())
nsets = max(2, min(8, int(3 * 126e6 // (2 * (M * K + K * N))) + 1))
sets = [(torch.randn(M, K, device="cuda", dtype=torch.float16), torch.randn(K, N, device="cuda", dtype=torch.float16))
        for _ in range(nsets)]
bias = torch.randn(N, device="cuda", dtype=torch.float16)
C = torch.empty(M, N, device="cuda", dtype=torch.float16)


def call(cfg, A, B):
    if cfg == "lt":
        return torch._addmm_activation(bias, A, B, out=C)
    if cfg == "cublas":
        return torch.matmul(A, B, out=C)
    if cfg == "auto":
        return ge.gemm_epilogue(A, B, bias, out=C)
    mc = 2 if cfg.endswith("m") else 1          # "512x2m": multicast clusters of two pairs
    bn, cg = (int(x) for x in cfg.rstrip("m").split("x"))
    return ge.gemm_epilogue(A, B, bias, out=C, tile_n=bn, cta_group=cg, multicast=mc)


flop = 2 * M * N * K
for cfg in cfgs:
    graphs = []
    per = 8
    for A, B in sets:
        call(cfg, A, B)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            for _ in range(per):
                call(cfg, A, B)
        graphs.append(g)
    for g in graphs: g.replay()
    torch.cuda.synchronize()
    t0 = time.perf_counter(); graphs[0].replay(); torch.cuda.synchronize(); dt = time.perf_counter() - t0
    reps = max(4, int(secs / max(dt, 1e-5)))
    samples, stop = [], threading.Event()

    def sampler():
        while not stop.is_set():
            samples.append((pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM),
                            pynvml.nvmlDeviceGetPowerUsage(h) / 1000.0))
            time.sleep(0.02)
    th = threading.Thread(target=sampler); th.start()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for i in range(reps): graphs[i % nsets].replay()
    e.record(); torch.cuda.synchronize()
    stop.set(); th.join()
    t = s.elapsed_time(e) * 1e-3 / (reps * per)
    sk = samples[len(samples) // 5:] or samples
    mhz = statistics.median(x[0] for x in sk); w = statistics.median(x[1] for x in sk)
    tf = flop / t / 1e12
    print(f"{M}x{N}x{K} {cfg:>7}: {tf:7.1f} TF/s  {t*1e6:8.1f} us  {mhz:5.0f} MHz  {w:5.0f} W  "
          f"{tf*1e12/(148*mhz*1e6):6.0f} flop/clk/SM  {tf/w:5.2f} TF/J", flush=True)
