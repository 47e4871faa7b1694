"""Dev tool: GPU time of one config from CUDA-graph replay (20 launches per graph, so host-side
call overhead is excluded); --eager times the Python call loop instead (host + GPU).
usage: timed.py M N K lay bn cg iters [--eager]"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2006_12645_b200 as ge
M, N, K = (int(x) for x in sys.argv[1:4]); lay = sys.argv[4]; bn, cg, it = (int(x) for x in sys.argv[5:8])
eager = "--eager" in sys.argv
A = torch.randn(M, K, device="cuda", dtype=torch.float16); B = torch.randn(K, N, device="cuda", dtype=torch.float16)
if lay[0] == "c": A = A.t().contiguous().t()
if lay[1] == "c": B = B.t().contiguous().t()
bias = torch.randn(N, device="cuda", dtype=torch.float16); C = torch.empty(M, N, device="cuda", dtype=torch.float16)
f = lambda: ge.gemm_epilogue(A, B, bias, out=C, tile_n=bn, cta_group=cg)
for _ in range(5): f()
torch.cuda.synchronize()
G = 20
if not eager:
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(G): f()
    g.replay(); torch.cuda.synchronize()
reps = max(1, it // G)
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
if eager:
    for _ in range(it): f()
    n = it
else:
    for _ in range(reps): g.replay()
    n = reps * G
e.record(); torch.cuda.synchronize()
t = s.elapsed_time(e) / n * 1e-3
print(f"{'eager' if eager else 'graph'} {2*M*N*K/t/1e12:.1f} TF/s  {t*1e6:.2f} us/launch over {n} launches")
