"""Dev tool: run one fused GEMM config a few times (for ncu captures).
usage: one_call.py M N K layouts tile_n cta_group [reps] [prologue] [batch]
Leading dimensions are padded to a multiple of 8 elements like bench.py (16-byte TMA pitch)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2006_12645_b200 as ge
M, N, K = (int(x) for x in sys.argv[1:4])
lay = sys.argv[4]; bn = int(sys.argv[5]); cg = int(sys.argv[6])
reps = int(sys.argv[7]) if len(sys.argv) > 7 else 3
pro = sys.argv[8] if len(sys.argv) > 8 and sys.argv[8] not in ("", "none") else None
batch = int(sys.argv[9]) if len(sys.argv) > 9 else 1
ld8 = lambda n: (n + 7) // 8 * 8


def operand(rows, cols, l):
    if l == "r":
        return torch.randn(batch, rows, ld8(cols), device="cuda", dtype=torch.float16)[:, :, :cols]
    return torch.randn(batch, cols, ld8(rows), device="cuda", dtype=torch.float16)[:, :, :rows].transpose(1, 2)


A = operand(M, K, lay[0])
B = operand(K, N, lay[1])
bias = torch.randn(N, device="cuda", dtype=torch.float16)
scale = torch.rand(K, device="cuda") + 0.5 if pro == "scale_k" else None
if pro == "hadamard":                  # the M x K tile S in A's layout
    scale = operand(M, K, lay[0])[0]
C = torch.empty(batch, M, ld8(N), device="cuda", dtype=torch.float16)[:, :, :N]
for _ in range(reps):
    if batch == 1:
        ge.gemm_epilogue(A[0], B[0], bias, tile_n=bn, cta_group=cg, prologue=pro, scale=scale, out=C[0])
    else:
        ge.gemm_epilogue_batched(A, B, bias, tile_n=bn, cta_group=cg, prologue=pro, scale=scale, out=C)
torch.cuda.synchronize()
print("ok", C.float().abs().mean().item(), ge.plan(M, N, K, batch=batch, layouts=lay, tile_n=bn, cta_group=cg,
                                                   prologue=pro))
