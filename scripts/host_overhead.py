"""Dev: host-side cost per call (tiny problem, so the GPU never limits): Python wrapper vs the raw
C-ABI call with prebuilt arguments vs torch/cuBLAS, microseconds per call."""
import ctypes, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2006_12645_b200 as ge
M = N = K = 128
A = torch.randn(M, K, device="cuda", dtype=torch.float16); B = torch.randn(K, N, device="cuda", dtype=torch.float16)
bias = torch.randn(N, device="cuda", dtype=torch.float16); C = torch.empty(M, N, device="cuda", dtype=torch.float16)
lib = ge.load_library()
o = ge._options("row", 0, None, None, torch.float16, 0, 0, 1, None)
sh = torch.cuda.current_stream().cuda_stream
raw = lambda: lib.gemm_epilogue(M, N, K, 0, 0, A.data_ptr(), K, B.data_ptr(), N, bias.data_ptr(), C.data_ptr(), N, 3, ctypes.byref(o), sh)
def bench(name, f, n=3000):
    for _ in range(50): f()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(n): f()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    print(f"{name:40s} {1e6 * (t1 - t) / n:7.2f} us/call (host)")
bench("ge.gemm_epilogue (python wrapper)", lambda: ge.gemm_epilogue(A, B, bias, out=C))
bench("ge.gemm_epilogue stream_k=1", lambda: ge.gemm_epilogue(A, B, bias, out=C, stream_k=1))
bench("raw C-ABI ctypes call", raw)
bench("torch._addmm_activation (cuBLASLt)", lambda: torch._addmm_activation(bias, A, B))
bench("torch.matmul", lambda: torch.matmul(A, B))
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    ge.gemm_epilogue(A, B, bias, out=C)
bench("graph replay (1 launch)", g.replay)
