"""Dev: stream-K on/off per shape (kernel time via events on back-to-back launches) + max error."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2006_12645_b200 as ge
shapes = [(1024, 1024, 1024), (2048, 2048, 2048), (4096, 4096, 4096), (5124, 700, 2048), (35, 8464, 2560)]
for (M, N, K) in shapes:
    A = torch.randn(M, K, device="cuda", dtype=torch.float16); B = torch.randn(K, N, device="cuda", dtype=torch.float16)
    bias = torch.randn(N, device="cuda", dtype=torch.float16)
    ref = torch.relu(torch.matmul(A.float(), B.float()) + bias.float())
    for cfg in [(256, 2), (256, 1), (128, 1)]:
        res = []
        for sk in (1, 2):
            try:
                pl = ge.plan(M, N, K, tile_n=cfg[0], cta_group=cfg[1], stream_k=sk)
                f = lambda: ge.gemm_epilogue(A, B, bias, tile_n=cfg[0], cta_group=cfg[1], stream_k=sk)
                C = f(); torch.cuda.synchronize()
                err = (C.float() - ref).abs().max().item()
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g):
                    for _ in range(10): f()
                g.replay(); torch.cuda.synchronize()
                s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                s.record(); [g.replay() for _ in range(5)]; e.record(); torch.cuda.synchronize()
                t = s.elapsed_time(e) / 50 * 1e-3
                res.append(f"sk={sk}({pl['stream_k_tiles']}): {2*M*N*K/t/1e12:7.1f} TF/s {t*1e6:7.1f}us err {err:.2f}")
            except Exception as ex:
                res.append(f"sk={sk}: ERR {str(ex)[:60]}")
        print((M, N, K), cfg, " | ".join(res), flush=True)
