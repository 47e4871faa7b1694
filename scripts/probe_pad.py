"""Dev probe: does the TMA store write past a ragged inner dimension (padding columns of C)?"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2006_12645_b200 as ge
torch.manual_seed(0)
for (M, N, K, swap, batch) in [(64, 1030, 136, 1, 1), (300, 1030, 136, 1, 1), (35, 1030, 136, 2, 1), (35, 1030, 136, 2, 3),
                               (35, 1030, 136, 1, 3), (300, 1027, 136, 1, 1)]:
    for dt in (torch.float16, torch.float32):
        A = torch.randint(-2, 3, (batch, M, K), device="cuda").half()
        Bp = torch.randint(-2, 3, (batch, K, 1040), device="cuda").half()
        B = Bp[:, :, :N]
        bias = torch.randint(-2, 3, (batch, N), device="cuda").half()
        Cbuf = torch.full((batch, M, 1040), -5.0, dtype=dt, device="cuda")
        ge.gemm_epilogue_batched(A, B, bias, out=Cbuf[:, :, :N], swap_ab=swap)
        torch.cuda.synchronize()
        ref = torch.relu(A.float() @ B.float() + bias.float()[:, None, :])
        pad_ok = bool((Cbuf[:, :, N:] == -5.0).all())
        bad_cols = sorted(set((Cbuf[:, :, N:] != -5.0).nonzero()[:, 2].tolist()))
        val_ok = bool((Cbuf[:, :, :N].float() == ref).all())
        print(M, N, K, "swap" if swap == 2 else "noswap", batch, dt, "pad_ok", pad_ok, "bad pad cols", [N + c for c in bad_cols][:8], "values_ok", val_ok, flush=True)
