"""Dev tool: GPU time per launch (CUDA-graph replay of 20 launches, operands L2-resident unless
--cold) for a list of shapes with the library selected by GE_LIBRARY_FILE; leading dimensions
padded to 8 elements like bench.py.
usage: timed_multi.py "M N K lay [bn cg]" ... [--iters N] [--cold] [--alt LAY2] [--tile-m 128|256] [--prologue scale_k] [--kw "swap_ab=1,stream_k=1"]
--alt LAY2: the graph alternates launches of layout `lay` and layout LAY2 (two kernel instantiations
back to back, like bench.py's multi-layout steps)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2006_12645_b200 as ge

alt = sys.argv[sys.argv.index("--alt") + 1] if "--alt" in sys.argv else None
tm = int(sys.argv[sys.argv.index("--tile-m") + 1]) if "--tile-m" in sys.argv else 0
pro = sys.argv[sys.argv.index("--prologue") + 1] if "--prologue" in sys.argv else None
extra = sys.argv[sys.argv.index("--kw") + 1] if "--kw" in sys.argv else ""
xkw = {k: int(v) for k, v in (x.split("=") for x in extra.split(",") if x)}
args = [a for a in sys.argv[1:] if not a.startswith("--") and a not in (alt, str(tm), pro, extra)]
iters = int(sys.argv[sys.argv.index("--iters") + 1]) if "--iters" in sys.argv else 400
if "--iters" in sys.argv:
    args.remove(str(iters))
cold = "--cold" in sys.argv
ld8 = lambda n: (n + 7) // 8 * 8
lib = os.path.basename(os.environ.get("GE_LIBRARY_FILE", "libgemm_epilogue.so"))


def operand(rows, cols, l, n):
    if l == "r":
        return [torch.randn(rows, ld8(cols), device="cuda", dtype=torch.float16)[:, :cols] for _ in range(n)]
    return [torch.randn(cols, ld8(rows), device="cuda", dtype=torch.float16)[:, :rows].t() for _ in range(n)]


for spec in args:
    f = spec.split()
    M, N, K = int(f[0]), int(f[1]), int(f[2])
    lay = f[3]
    bn, cg = (int(f[4]), int(f[5])) if len(f) > 5 else (0, 0)
    nset = max(1, min(16, int(3 * 126e6 // max(1, 2 * (M * K + K * N))))) if cold else 1
    As, Bs = operand(M, K, lay[0], nset), operand(K, N, lay[1], nset)
    if alt:                      # odd launches use the second layout
        As2, Bs2 = operand(M, K, alt[0], nset), operand(K, N, alt[1], nset)
        As = [x for pair in zip(As, As2) for x in pair]
        Bs = [x for pair in zip(Bs, Bs2) for x in pair]
        nset *= 2
    bias = torch.randn(N, device="cuda", dtype=torch.float16)
    C = torch.empty(M, ld8(N), device="cuda", dtype=torch.float16)[:, :N]
    scale = (torch.rand(K, device="cuda") + 0.5) if pro == "scale_k" else None
    if pro == "hadamard":          # the M x K tile S in A's layout
        scale = operand(M, K, lay[0], 1)[0]
    kw = dict(prologue=pro, scale=scale) if pro else {}
    kw.update(xkw)
    G = 20
    for i in range(3):
        ge.gemm_epilogue(As[i % nset], Bs[i % nset], bias, out=C, tile_n=bn, cta_group=cg, tile_m=tm, **kw)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for i in range(G):
            ge.gemm_epilogue(As[i % nset], Bs[i % nset], bias, out=C, tile_n=bn, cta_group=cg, tile_m=tm, **kw)
    g.replay()
    torch.cuda.synchronize()
    reps = max(1, iters // G)
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        g.replay()
    e.record()
    torch.cuda.synchronize()
    t = s.elapsed_time(e) / (reps * G) * 1e-3
    pl = ge.plan(M, N, K, layouts=lay, tile_n=bn, cta_group=cg, tile_m=tm, prologue=pro, **xkw)
    if alt:
        spec = spec + "/" + alt
    if extra:
        spec = spec + " " + extra
    print(f"{lib:28s} {spec:26s} {t * 1e6:8.2f} us {2 * M * N * K / t / 1e12:7.1f} TF/s  "
          f"plan {pl['tile_m']}x{pl['tile_n']} cg{pl['cta_group']} split{pl['split_k']} swap{pl['swap_ab']}", flush=True)
