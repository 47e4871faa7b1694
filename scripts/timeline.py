"""Dev tool: per-launch %globaltimer timeline of CTA 0 for graph-replayed back-to-back launches
(diagnostics build, GE_LIBRARY_FILE=.../libgemm_epilogue_dbg.so, GE_DEBUG_STATS unset so no
per-launch counter reset breaks the PDL overlap).  usage: timeline.py "M N K lay [bn cg]" ... [--kw a=1]"""
import ctypes
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2006_12645_b200 as ge

extra = sys.argv[sys.argv.index("--kw") + 1] if "--kw" in sys.argv else ""
xkw = {k: int(v) for k, v in (x.split("=") for x in extra.split(",") if x)}
specs = [a for a in sys.argv[1:] if not a.startswith("--") and a != extra]
ld8 = lambda n: (n + 7) // 8 * 8
lib = ge.load_library()
lib.ge_debug_set_timeline.argtypes = [ctypes.c_void_p]
NAMES = ["entry", "setup", "wait", "first_full", "last_commit", "epi_tfull", "epi_end", "teardown", "exit",
         "prod_first", "prod_last"]


def operand(rows, cols, l, n):
    if l == "r":
        return [torch.randn(rows, ld8(cols), device="cuda", dtype=torch.float16)[:, :cols] for _ in range(n)]
    return [torch.randn(cols, ld8(rows), device="cuda", dtype=torch.float16)[:, :rows].t() for _ in range(n)]


for spec in specs:
    f = spec.split()
    M, N, K, lay = int(f[0]), int(f[1]), int(f[2]), f[3]
    bn, cg = (int(f[4]), int(f[5])) if len(f) > 5 else (0, 0)
    nset = max(1, min(16, int(3 * 126e6 // max(1, 2 * (M * K + K * N)))))
    As, Bs = operand(M, K, lay[0], nset), operand(K, N, lay[1], nset)
    bias = torch.randn(N, device="cuda", dtype=torch.float16)
    C = torch.empty(M, ld8(N), device="cuda", dtype=torch.float16)[:, :N]
    G = 20
    buf = torch.zeros(1 + 24 * 64, dtype=torch.int64, device="cuda")
    lib.ge_debug_set_timeline(ctypes.c_void_p(buf.data_ptr()))
    call = lambda i: ge.gemm_epilogue(As[i % nset], Bs[i % nset], bias, out=C, tile_n=bn, cta_group=cg, **xkw)
    for i in range(3):
        call(i)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for i in range(G):
            call(i)
    buf.zero_()
    torch.cuda.synchronize()
    g.replay()
    torch.cuda.synchronize()
    lib.ge_debug_set_timeline(ctypes.c_void_p(0))
    n = int(buf[0].item())
    t = buf[1:1 + 24 * n].view(n, 24).cpu().tolist()
    pl = ge.plan(M, N, K, layouts=lay, tile_n=bn, cta_group=cg, **xkw)
    print(f"== {spec} {extra}  plan {pl['tile_m']}x{pl['tile_n']} cg{pl['cta_group']} split{pl['split_k']} "
          f"swap{pl['swap_ab']}  launches {n}")
    print("  (ns, relative to this launch's entry; gap = entry - previous exit)")
    print("   i    gap  setup   wait  pfirst  full1  lastc  tfull  eend  tdown  exit  plast decode barini expect  loadA  alloc  wseq policy")
    rows = []
    for i in range(n):
        r = t[i]
        e = r[0]
        gap = e - t[i - 1][8] if i > 0 else 0
        rel = [r[k] - e if r[k] else -1 for k in (1, 2, 9, 3, 4, 5, 6, 7, 8, 10, 11, 12, 13, 14, 15, 16, 17)]
        rows.append([gap] + rel)
        print(f"  {i:2d} {gap:6d} " + " ".join(f"{x:6d}" for x in rel))
    import statistics
    med = [statistics.median(c) for c in zip(*rows[2:])]
    print("  med " + " ".join(f"{x:6.0f}" for x in med))
    print(f"  entry-to-entry median {statistics.median([t[i][0] - t[i-1][0] for i in range(1, n)]):.0f} ns")
