"""Dev tool: one cuBLASLt fused bias+ReLU call (torch._addmm_activation), for ncu captures.
usage: lt_call.py M N K [reps]"""
import sys, torch
M, N, K = (int(x) for x in sys.argv[1:4])
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 1
A = torch.randn(M, K, device="cuda", dtype=torch.float16); B = torch.randn(K, N, device="cuda", dtype=torch.float16)
bias = torch.randn(N, device="cuda", dtype=torch.float16)
for _ in range(reps):
    C = torch._addmm_activation(bias, A, B)
torch.cuda.synchronize()
print("ok", C.float().abs().mean().item())
