"""Multi-GPU sharding of independent GEMMs.

The fused GEMM has no exchange step: output tiles and batch items are independent (the paper is
single-GPU).  So the data path shards with NO collective:

* batched problems split the batch into contiguous blocks, rank r owning items
  [r*B/P, (r+1)*B/P) (remainders spread over the first ranks);
* a single large GEMM splits M into row blocks cut at multiples of the 256-row tile, so every rank
  runs exactly the tiles the 1-GPU launch would (bitwise-identical results); A is sliced by rows,
  B and bias are replicated, and each rank's C rows are contiguous in row-major C.

A collective appears only when the caller asks for the full output on every rank
(``gather=True``): one NCCL all-gather of the row/batch blocks over NVLink/NVSwitch, off the hot
path.  All functions take ``torch.distributed`` state from the default process group.
"""
from __future__ import annotations

from typing import Optional

import torch
import torch.distributed as dist

ROW_QUANTUM = 256       # tile height of the CTA-pair kernel: M cuts at multiples keep tiles identical


def shard_range(n: int, rank: int, world: int, quantum: int = 1) -> tuple[int, int]:
    """Contiguous [lo, hi) block of n units owned by `rank`, cut at multiples of `quantum`
    (the last rank takes the ragged tail).  Blocks are balanced to within one quantum."""
    if world <= 0 or not (0 <= rank < world):
        raise ValueError("bad rank/world")
    q = max(1, quantum)
    units = (n + q - 1) // q
    base, rem = divmod(units, world)
    lo_u = rank * base + min(rank, rem)
    hi_u = lo_u + base + (1 if rank < rem else 0)
    return min(n, lo_u * q), min(n, hi_u * q)


def all_ranges(n: int, world: int, quantum: int = 1) -> list[tuple[int, int]]:
    return [shard_range(n, r, world, quantum) for r in range(world)]


def _world():
    if dist.is_available() and dist.is_initialized():
        return dist.get_rank(), dist.get_world_size()
    return 0, 1


def gather_rows(local: torch.Tensor, n_total: int, quantum: int = 1) -> torch.Tensor:
    """All-gather row blocks (dim 0) of possibly unequal size into the full tensor on every rank.
    Blocks are padded to the largest block for the collective and trimmed afterwards."""
    rank, world = _world()
    if world == 1:
        return local
    ranges = all_ranges(n_total, world, quantum)
    cap = max(hi - lo for lo, hi in ranges)
    pad = torch.zeros((cap,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    pad[: local.shape[0]] = local
    buf = torch.empty((world * cap,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    dist.all_gather_into_tensor(buf, pad)
    parts = [buf[r * cap: r * cap + (hi - lo)] for r, (lo, hi) in enumerate(ranges)]
    return torch.cat(parts, dim=0)


def sharded_gemm_epilogue_batched(A: torch.Tensor, B: torch.Tensor, bias: Optional[torch.Tensor] = None, *,
                                  gather: bool = False, compute=None, **kw) -> torch.Tensor:
    """Rank-local slice of a batched GEMM+epilogue.  A (b, M, K), B (b, K, N) and a per-item bias
    (b, N) may be given either in full (each rank slices its items) or already sliced
    (``kw['presliced']=True``).  Returns this rank's C items, or all items if gather=True.
    ``compute`` overrides the per-rank kernel call (tests on CPU use the oracle)."""
    from . import gemm_epilogue_batched
    presliced = kw.pop("presliced", False)
    total = kw.pop("total_batch", A.shape[0])
    rank, world = _world()
    lo, hi = shard_range(total, rank, world)
    if not presliced:
        A, B = A[lo:hi], B[lo:hi]
        if bias is not None and bias.dim() == 2:
            bias = bias[lo:hi]
    fn = compute or gemm_epilogue_batched
    C = fn(A, B, bias, **kw) if hi > lo else torch.empty((0, A.shape[1], B.shape[2]), dtype=torch.float16,
                                                         device=A.device)
    return gather_rows(C, total) if gather else C


def sharded_gemm_epilogue_rows(A: torch.Tensor, B: torch.Tensor, bias: Optional[torch.Tensor] = None, *,
                               gather: bool = False, compute=None, **kw) -> torch.Tensor:
    """Row-block (M) shard of one GEMM: rank r computes rows shard_range(M, r, P, 256) of C.
    A is the full (M, K) operand or the rank's row block (``presliced=True``); B, bias replicated
    (a COL bias is sliced with A)."""
    from . import gemm_epilogue
    presliced = kw.pop("presliced", False)
    M = kw.pop("total_rows", A.shape[0])
    rank, world = _world()
    lo, hi = shard_range(M, rank, world, ROW_QUANTUM)
    if not presliced:
        A = A[lo:hi]
        if bias is not None and kw.get("bias_mode") == "col":
            bias = bias[lo:hi]
    fn = compute or gemm_epilogue
    C = fn(A, B, bias, **kw) if hi > lo else torch.empty((0, B.shape[1]), dtype=torch.float16, device=A.device)
    return gather_rows(C, M, ROW_QUANTUM) if gather else C
