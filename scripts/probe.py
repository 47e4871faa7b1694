"""Quick perf probe (dev tool): TFLOP/s of the fused kernel per config vs torch (cuBLAS) + add + relu."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2006_12645_b200 as ge

def timeit(fn, iters=20, warm=5):
    for _ in range(warm): fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(iters): fn()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / iters * 1e-3

sizes = [int(x) for x in (sys.argv[1].split(",") if len(sys.argv) > 1 else ["4096", "8192"])]
cfgs = [(256, 1), (128, 1), (256, 2), (128, 2)]
for n in sizes:
    M = N = K = n
    A = torch.randn(M, K, device="cuda", dtype=torch.float16)
    B = torch.randn(K, N, device="cuda", dtype=torch.float16)
    bias = torch.randn(N, device="cuda", dtype=torch.float16)
    fl = 2 * M * N * K
    t = timeit(lambda: torch.relu_(torch.matmul(A, B).add_(bias)))
    t2 = timeit(lambda: torch.matmul(A, B))
    print(f"{n}^3 torch unfused {fl/t/1e12:7.1f} TF/s   cublas matmul only {fl/t2/1e12:7.1f}", flush=True)
    for lay in ("rr", "rc", "cr", "cc"):
        Aa = A if lay[0] == "r" else A.t().contiguous().t()
        Bb = B if lay[1] == "r" else B.t().contiguous().t()
        ref = torch.relu(torch.matmul(A, B).float() + bias.float())
        for bn, cg in cfgs:
            try:
                C = ge.gemm_epilogue(Aa, Bb, bias, tile_n=bn, cta_group=cg)
                torch.cuda.synchronize()
                err = (C.float() - ref).abs().max().item()
                t = timeit(lambda: ge.gemm_epilogue(Aa, Bb, bias, tile_n=bn, cta_group=cg))
                print(f"  {lay} bn={bn} cg={cg}: {fl/t/1e12:7.1f} TF/s  {t*1e6:8.1f} us  maxerr {err:.3g}", flush=True)
            except Exception as ex:
                print(f"  {lay} bn={bn} cg={cg}: ERROR {ex}", flush=True)
                raise
