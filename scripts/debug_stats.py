"""Dev tool: per-role blocked cycles (GE_DEBUG_STATS=1) of one config. usage: M N K lay bn cg"""
import os, sys
os.environ["GE_DEBUG_STATS"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2006_12645_b200 as ge
M, N, K = (int(x) for x in sys.argv[1:4]); lay = sys.argv[4]; bn, cg = int(sys.argv[5]), int(sys.argv[6])
sk = int(sys.argv[7]) if len(sys.argv) > 7 else 0
mc = int(sys.argv[8]) if len(sys.argv) > 8 else 0
pro = sys.argv[9] if len(sys.argv) > 9 else None
ld8 = lambda n: (n + 7) // 8 * 8          # padded leading dimensions (16-byte TMA pitch), like bench.py
def operand(rows, cols, l):
    if l == "r":
        return torch.randn(rows, ld8(cols), device="cuda", dtype=torch.float16)[:, :cols]
    return torch.randn(cols, ld8(rows), device="cuda", dtype=torch.float16)[:, :rows].t()
A = operand(M, K, lay[0]); B = operand(K, N, lay[1])
bias = torch.randn(N, device="cuda", dtype=torch.float16)
C = torch.empty(M, ld8(N), device="cuda", dtype=torch.float16)[:, :N]
scale = (torch.rand(K, device="cuda") + 0.5) if pro == "scale_k" else None
for _ in range(20): ge.gemm_epilogue(A, B, bias, out=C, tile_n=bn, cta_group=cg, stream_k=sk, multicast=mc,
                                     prologue=pro, scale=scale)
torch.cuda.synchronize()
st = ge.debug_stats()
lead = [s for i, s in enumerate(st) if (cg == 1 or i % 2 == 0) and s["total"] > 0]   # active leaders
def avg(k, rows): return sum(r[k] for r in rows) / max(1, len(rows))
tot = avg("total", lead)
print(f"{M}x{N}x{K} {lay} bn={bn} cg={cg}: total {tot:.0f} cyc/CTA(leader)")
for k in ("prod_wait_empty", "mma_wait_full", "mma_wait_tempty", "epi_wait_tfull", "epi_to_release0", "epi_to_release1", "epi_tile", "epi_tmem_ld", "epi_math", "sk_owner_wait", "sk_partial_write", "sk_pieces", "epi_end"):
    print(f"  {k:18s} {avg(k, lead):12.0f} cyc  ({100*avg(k, lead)/tot:5.1f}% of total)")
print("  prologue transform (sum over its 4 warps): wait for stage", avg("xf_wait", lead), " rewrite", avg("xf_work", lead))
print("  MMA warp: issue", avg("mma_issue", lead), " commits", avg("mma_commit", lead))
print("  producer: issue", avg("prod_issue", lead), " wait empty", avg("prod_wait_empty", lead), " loop total", avg("prod_total", lead))
# split-K epilogue phases (per warp lane 0, summed over the CTA's epilogue warps)
print("  split-K owner phases (sum over warps): tmem ld", avg("own_ld", lead), " add", avg("own_add", lead),
      " math", avg("own_math", lead), " store", avg("own_st", lead))
print("  split-K: sends (sum over warps)", avg("epi_tmem_ld", lead), " owner compute+store (sum over warps)", avg("epi_math", lead))
print("  per-CTA mma_wait_full min/max:", min(r["mma_wait_full"] for r in lead), max(r["mma_wait_full"] for r in lead))

ends = sorted(r["epi_end"] for r in st)
print("  epi_end per CTA: min", ends[0], "median", ends[len(ends)//2], "max", ends[-1])
tots = sorted(r["total"] for r in lead)
print("  mma end (total) per leader: min", tots[0], "median", tots[len(tots)//2], "max", tots[-1])
print("  slowest CTAs (idx: epi_end, mma_end(total), owner_wait, partial_write, pieces, epi_tile):")
for i, r in sorted(enumerate(st), key=lambda x: -x[1]["epi_end"])[:6]:
    print(f"    {i:3d}: {r['epi_end']:7d} {r['total']:7d} {r['sk_owner_wait']:7d} {r['sk_partial_write']:6d} {r['sk_pieces']} {r['epi_tile']:7d}")
fm = sorted(r["first_mma"] for r in lead)
print("  first MMA (cycles after kernel start) per leader: min", fm[0], "median", fm[len(fm)//2], "max", fm[-1])

# absolute timeline (%globaltimer, ns) across CTAs: launch stagger, setup, epilogue end, exit
ent = [r["g_entry"] for r in st if r["g_entry"]]
if ent:
    t0 = min(ent)
    rel = lambda k: sorted(r[k] - t0 for r in st if r[k])
    for k in ("g_entry", "g_start", "g_epi_end", "g_exit"):
        v = rel(k)
        if v:
            print(f"  {k:10s} ns after first entry: min {v[0]:7d} median {v[len(v)//2]:7d} max {v[-1]:7d} (n={len(v)})")
