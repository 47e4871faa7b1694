"""Dev: measured TF/s of every kernel configuration per shape (CUDA-graph timed, rotating operands),
plus what the heuristic picks.  Output feeds config_eff / the plan cost model."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2006_12645_b200 as ge
shapes = [(1024, 1024, 1024), (2048, 2048, 2048), (4096, 4096, 4096), (8192, 8192, 8192), (5124, 704, 2048),
          (35, 8464, 2560), (2048, 2048, 8192), (512, 512, 512), (3072, 3072, 3072), (6144, 6144, 6144),
          (3840, 2560, 3584), (1536, 3456, 3584), (4096, 4096, 8192)]
RC = "--rc" in sys.argv          # column-major (K-major) B: the paper's rc layout
args = [a for a in sys.argv[1:] if a != "--rc"]
if args:
    shapes = [tuple(int(x) for x in s.split("x")) for s in args]
# (tile_n, cta_group, multicast): multicast 2 = clusters of two CTA pairs sharing B
cfgs = [(512, 2, 1), (256, 2, 1), (512, 2, 2), (256, 2, 2), (256, 1, 1), (192, 2, 1), (192, 1, 1), (128, 2, 1), (128, 1, 1), (64, 1, 1)]
res = {}
for (M, N, K) in shapes:
    nsets = max(1, min(16, int(3 * 126e6 // (2 * (M * K + K * N))) + 1))
    sets = [(torch.randn(M, K, device="cuda", dtype=torch.float16),
             torch.randn(N, K, device="cuda", dtype=torch.float16).t() if RC else
             torch.randn(K, N, device="cuda", dtype=torch.float16)) for _ in range(nsets)]
    bias = torch.randn(N, device="cuda", dtype=torch.float16)
    C = torch.empty(M, N, device="cuda", dtype=torch.float16)
    row = {}
    for bn, cg, mc in cfgs + [(0, 0, 0)]:
        if bn == 192 and cg == 2 and not RC:
            continue
        graphs = []
        for A, B in sets:
            ge.gemm_epilogue(A, B, bias, out=C, tile_n=bn, cta_group=cg, multicast=mc)
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                for _ in range(4):
                    ge.gemm_epilogue(A, B, bias, out=C, tile_n=bn, cta_group=cg, multicast=mc)
            graphs.append(g)
        for g in graphs[:3]: g.replay()
        torch.cuda.synchronize()
        it = max(8, min(200, int(2e-1 / (2 * M * N * K / 1.2e15) / 4)))
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for i in range(it): graphs[i % nsets].replay()
        e.record(); torch.cuda.synchronize()
        t = s.elapsed_time(e) / (it * 4) * 1e-3
        row["auto" if bn == 0 else f"{bn}x{cg}" + ("m" if mc == 2 else "")] = round(2 * M * N * K / t / 1e12, 1)
    pl = ge.plan(M, N, K, layouts="rc" if RC else "rr")
    row["auto_pick"] = f"{pl['tile_n']}x{pl['cta_group']}" + ("m" if pl["tile_m"] == 512 else "")
    res[f"{M}x{N}x{K}"] = row
    print(f"{M}x{N}x{K}", row, flush=True)
json.dump(res, open("gpurun_out/tune_sweep.json", "w"), indent=1)
