"""Dev: split-K (auto plan) vs data-parallel (stream_k=1) GPU time via CUDA-graph replay."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2006_12645_b200 as ge
SH = [(640, 1024, 3840), (2048, 128, 3456), (384, 768, 1536), (128, 2176, 3200), (1024, 1536, 3840),
      (768, 1024, 3456), (1920, 384, 3200), (384, 896, 3200), (3072, 128, 3968), (2560, 128, 2816)]
def t(f, it=20):
    f(); torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(it): f()
    g.replay(); torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(); [g.replay() for _ in range(5)]; e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / (5 * it) * 1e-3
for (M, N, K) in SH:
    A = torch.randn(M, K, device="cuda", dtype=torch.float16); B = torch.randn(N, K, device="cuda", dtype=torch.float16).t()
    bias = torch.randn(N, device="cuda", dtype=torch.float16); C = torch.empty(M, N, device="cuda", dtype=torch.float16)
    p = ge.plan(M, N, K, layouts="rc")
    ts = t(lambda: ge.gemm_epilogue(A, B, bias, out=C))
    td = t(lambda: ge.gemm_epilogue(A, B, bias, out=C, stream_k=1))
    tl = t(lambda: torch._addmm_activation(bias, A, B))
    f = 2 * M * N * K
    print(f"{M}x{N}x{K} plan {p['tile_n']}x{p['cta_group']} split {p['split_k']}: auto {f/ts/1e12:6.1f} TF/s ({ts*1e6:5.1f} us)"
          f"  dp {f/td/1e12:6.1f} ({td*1e6:5.1f} us)  cublaslt {f/tl/1e12:6.1f} ({tl*1e6:5.1f} us)", flush=True)
