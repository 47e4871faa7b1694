"""Per-call time (us) of our kernel in one CUDA graph of R calls, for a few tiny/small shapes (rc).
Run under different GE_DEBUG_FLAGS / GE_DEBUG_NOLOAD / GE_PDL settings to attribute fixed costs."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2006_12645_b200 as ge
R = 40
out = []
for (M, N, K) in [(128, 64, 64), (512, 128, 512), (1152, 256, 128), (640, 2048, 1408), (2048, 2048, 2048)]:
    A = torch.randn(M, K, device="cuda", dtype=torch.float16)
    B = torch.randn(N, K, device="cuda", dtype=torch.float16).t()
    bias = torch.randn(N, device="cuda", dtype=torch.float16)
    C = torch.empty(M, N, device="cuda", dtype=torch.float16)
    ge.gemm_epilogue(A, B, bias, out=C)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(R):
            ge.gemm_epilogue(A, B, bias, out=C)
    g.replay(); torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(5):
        g.replay()
    e.record(); torch.cuda.synchronize()
    out.append(f"{M}x{N}x{K}:{s.elapsed_time(e) / (5 * R) * 1e3:.2f}")
print(os.environ.get("TAG", ""), " ".join(out), flush=True)
