"""Dev tool: cuBLAS / cuBLASLt comparators at one shape, sustained (back-to-back) timing."""
import sys, torch
M = N = K = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
it = int(sys.argv[2]) if len(sys.argv) > 2 else 200
A = torch.randn(M, K, device="cuda", dtype=torch.float16); B = torch.randn(K, N, device="cuda", dtype=torch.float16)
bias = torch.randn(N, device="cuda", dtype=torch.float16)
for name, f in [("matmul", lambda: torch.matmul(A, B)), ("addmm_relu(cublasLt epi)", lambda: torch._addmm_activation(bias, A, B)),
                ("unfused", lambda: torch.relu_(torch.matmul(A, B).add_(bias)))]:
    for _ in range(10): f()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(it): f()
    e.record(); torch.cuda.synchronize()
    t = s.elapsed_time(e) / it * 1e-3
    print(f"{name}: sustained {2*M*N*K/t/1e12:.1f} TF/s ({t*1e6:.1f} us)")
