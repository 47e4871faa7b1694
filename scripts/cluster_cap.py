"""Dev: co-resident split-K clusters per (tile_n, S) as the planner sees them, plus plans."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2006_12645_b200 as ge
A = torch.randn(256, 256, device="cuda", dtype=torch.float16)
ge.gemm_epilogue(A, A, torch.zeros(256, device="cuda", dtype=torch.float16)); torch.cuda.synchronize()
