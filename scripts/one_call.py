"""Dev tool: run one fused GEMM config a few times (for ncu captures).
usage: one_call.py M N K layouts tile_n cta_group [reps] [prologue]"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2006_12645_b200 as ge
M, N, K = (int(x) for x in sys.argv[1:4])
lay = sys.argv[4]; bn = int(sys.argv[5]); cg = int(sys.argv[6])
reps = int(sys.argv[7]) if len(sys.argv) > 7 else 3
pro = sys.argv[8] if len(sys.argv) > 8 else None
A = torch.randn(M, K, device="cuda", dtype=torch.float16)
B = torch.randn(K, N, device="cuda", dtype=torch.float16)
if lay[0] == "c": A = A.t().contiguous().t()
if lay[1] == "c": B = B.t().contiguous().t()
bias = torch.randn(N, device="cuda", dtype=torch.float16)
scale = torch.rand(K, device="cuda") + 0.5 if pro == "scale_k" else None
for _ in range(reps):
    C = ge.gemm_epilogue(A, B, bias, tile_n=bn, cta_group=cg, prologue=pro, scale=scale)
torch.cuda.synchronize()
print("ok", C.float().abs().mean().item())
