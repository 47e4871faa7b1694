"""Dev: throughput of the widened features (pointwise ops, sum of matmuls) vs plain bias+ReLU."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2006_12645_b200 as ge

def timed(fn, it=20):
    fn(); g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(4): fn()
    g.replay(); torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(); [g.replay() for _ in range(it)]; e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / (it * 4) * 1e-3

out = {}
M = N = K = 4096
A = torch.randn(M, K, device="cuda", dtype=torch.float16); B = torch.randn(K, N, device="cuda", dtype=torch.float16)
P = torch.randn(M, K, device="cuda", dtype=torch.float16); Q = torch.randn(K, N, device="cuda", dtype=torch.float16)
bias = torch.randn(N, device="cuda", dtype=torch.float16); C = torch.empty(M, N, device="cuda", dtype=torch.float16)
fl = 2.0 * M * N * K
for op in ("bias_relu", "bias_sigmoid", "bias_tanh", "sub_bias_relu"):
    t = timed(lambda: ge.gemm_epilogue(A, B, bias, op=op, out=C))
    out[f"4096^3 {op}"] = round(fl / t / 1e12, 1)
t = timed(lambda: ge.gemm2_epilogue(A, B, P, Q, bias, out=C))
out["4096^3 gemm2 (A.B+P.Q)+bias+relu"] = round(2 * fl / t / 1e12, 1)
t = timed(lambda: torch.relu_(torch.matmul(A, B).add_(torch.matmul(P, Q)).add_(bias)))
out["4096^3 unfused torch A@B + P@Q + bias, relu"] = round(2 * fl / t / 1e12, 1)
t = timed(lambda: torch.relu_(torch.addmm(bias, torch.cat([A, P], 1), torch.cat([B, Q], 0))))
out["4096^3 torch cat-K addmm + relu (incl. cats)"] = round(2 * fl / t / 1e12, 1)
print(json.dumps(out, indent=1))
json.dump(out, open("gpurun_out/feature_perf.json", "w"), indent=1)
