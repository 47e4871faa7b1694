"""Dev: small shapes through every kernel configuration, for compute-sanitizer runs."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2006_12645_b200 as ge
torch.manual_seed(0)
for (M, N, K) in [(300, 520, 200), (129, 257, 65)]:
    up8 = lambda v: (v + 7) // 8 * 8                       # TMA: 16-byte row pitch
    A = torch.randn(M, up8(K), device="cuda", dtype=torch.float16)[:, :K]
    B = torch.randn(N, up8(K), device="cuda", dtype=torch.float16)[:, :K].t()
    bias = torch.randn(N, device="cuda", dtype=torch.float16)
    scale = torch.rand(K, device="cuda") + 0.5
    for bn, cg in [(512, 2), (256, 2), (192, 2), (256, 1), (192, 1), (128, 2), (128, 1), (64, 1)]:
        for sk in (1, 2):
            ge.gemm_epilogue(A, B, bias, tile_n=bn, cta_group=cg, stream_k=sk)
        ge.gemm_epilogue(A, B, bias, tile_n=bn, cta_group=cg, prologue="scale_k", scale=scale, stream_k=1)
        ge.gemm_epilogue(A, B, bias, tile_n=bn, cta_group=cg, out_dtype=torch.float32, stream_k=1)
        ge.gemm_epilogue(A, B, bias, tile_n=bn, cta_group=cg, op="literal_bias_relu", stream_k=1)
    # multicast clusters of two CTA pairs (B tiles multicast to both pairs), both tile widths
    for bn in (512, 256):
        ge.gemm_epilogue(A, B, bias, tile_n=bn, cta_group=2, multicast=2)
        ge.gemm_epilogue(A, B, bias, tile_n=bn, cta_group=2, multicast=2, out_dtype=torch.float32)
    # round 2: half-row CTA pairs, swap-AB (skinny, transposed store), Hadamard prologue, all layouts
    S = (torch.rand(M, up8(K), device="cuda") + 0.5).half()[:, :K]
    for bn in (128, 256):
        ge.gemm_epilogue(A, B, bias, tile_n=bn, cta_group=2, tile_m=128)
        ge.gemm_epilogue(A, B, bias, tile_n=bn, cta_group=2, tile_m=128, out_dtype=torch.float32)
    ge.gemm_epilogue(A, B, bias, prologue="hadamard", scale=S, stream_k=1)
    ge.gemm_epilogue(A, B, bias, prologue="hadamard", scale=S, tile_n=512, cta_group=2)
    ge.gemm_epilogue(A[:35], B, bias, swap_ab=2)
    Acr = torch.empty(K, up8(M), device="cuda", dtype=torch.float16)[:, :M]       # column-major A, padded ld
    Acr.copy_(A.t())
    Brr = torch.empty(K, up8(N), device="cuda", dtype=torch.float16)[:, :N]       # row-major B, padded ld
    Brr.copy_(B)
    ge.gemm_epilogue(Acr.t(), Brr, bias, tile_n=256, cta_group=2)                  # cr, runtime layouts
    # split-K clusters (DSMEM reduce-scatter): a long-K shape the planner splits
    A2 = torch.randn(256, 64 * 40, device="cuda", dtype=torch.float16)
    B2 = torch.randn(64 * 40, 256, device="cuda", dtype=torch.float16)
    b2 = torch.randn(256, device="cuda", dtype=torch.float16)
    ge.gemm_epilogue(A2, B2, b2)
torch.cuda.synchronize()
print("sanitize workload done")
