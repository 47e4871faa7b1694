"""Dev tool: sustained timing (back-to-back launches) of one config. usage: timed.py M N K lay bn cg iters"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2006_12645_b200 as ge
M, N, K = (int(x) for x in sys.argv[1:4]); lay = sys.argv[4]; bn, cg, it = (int(x) for x in sys.argv[5:8])
A = torch.randn(M, K, device="cuda", dtype=torch.float16); B = torch.randn(K, N, device="cuda", dtype=torch.float16)
if lay[0] == "c": A = A.t().contiguous().t()
if lay[1] == "c": B = B.t().contiguous().t()
bias = torch.randn(N, device="cuda", dtype=torch.float16); C = torch.empty(M, N, device="cuda", dtype=torch.float16)
f = lambda: ge.gemm_epilogue(A, B, bias, out=C, tile_n=bn, cta_group=cg)
for _ in range(10): f()
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(it): f()
e.record(); torch.cuda.synchronize()
t = s.elapsed_time(e) / it * 1e-3
print(f"sustained {2*M*N*K/t/1e12:.1f} TF/s  {t*1e6:.1f} us/launch over {it} launches")
