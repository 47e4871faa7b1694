"""Dev: run cuBLASLt fused bias+ReLU (torch._addmm_activation) and our kernel once per shape, for an
ncu launch list (kernel names, grid, cluster, time).  usage: ncu ... python scripts/cublas_names.py"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2006_12645_b200 as ge
SHAPES = [(3840, 2560, 3584), (640, 1024, 3840), (2048, 128, 3456), (1920, 384, 3200), (384, 768, 1536),
          (768, 1024, 3456), (1536, 3456, 3584), (1664, 1664, 3712), (128, 2176, 3200), (2816, 384, 2432)]
for (M, N, K) in SHAPES:
    A = torch.randn(M, K, device="cuda", dtype=torch.float16)
    B = torch.randn(N, K, device="cuda", dtype=torch.float16).t()
    bias = torch.randn(N, device="cuda", dtype=torch.float16)
    torch.cuda.nvtx.range_push(f"{M}x{N}x{K}")
    torch._addmm_activation(bias, A, B)
    ge.gemm_epilogue(A, B, bias)
    torch.cuda.synchronize()
    torch.cuda.nvtx.range_pop()
    print(M, N, K, ge.plan(M, N, K, layouts="rc"), flush=True)
