"""Multi-GPU sharding of independent GEMMs.

The fused GEMM has no exchange step: output tiles and batch items are independent (the paper is
single-GPU).  So the data path shards with NO collective:

* batched problems split the batch into contiguous blocks, rank r owning items
  [r*B/P, (r+1)*B/P) (remainders spread over the first ranks);
* a single large GEMM splits M into row blocks cut at multiples of the 256-row tile; A is sliced by
  rows, B and a row bias are replicated (a column or full bias is sliced with A's rows), and each
  rank's C rows are contiguous in row-major C.

Per rank the fused kernel computes exactly the definition on its slice, so shards always agree
with the 1-GPU result within the north_star bound.  They agree BITWISE when every rank's launch
runs the same tile configuration with no split or stream-K reduction (a smaller per-rank problem
can change the planner's choice and with it the fp32 summation order, DESIGN.md R-C13): pass
``stream_k=1`` and an explicit ``tile_n``/``cta_group`` to pin it.

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
        bias = _slice_bias_items(bias, kw.get("bias_mode", "row"), lo, hi)
    fn = compute or gemm_epilogue_batched
    C = fn(A, B, bias, **kw) if hi > lo else torch.empty((0, A.shape[1], B.shape[2]),
                                                         dtype=kw.get("out_dtype", torch.float16), device=A.device)
    return gather_rows(C, total) if gather else C


def _slice_bias_items(bias, bias_mode, lo, hi):
    """Per-item biases are sliced to the rank's items; a bias shared by every item is passed as is:
    row/col: (b, L) per item vs (L,) shared; full: (b, M, ld) per item vs (M, ld) shared."""
    if bias is None:
        return None
    per_item = bias.dim() == (3 if bias_mode == "full" else 2)
    return bias[lo:hi] if per_item else bias


def sharded_gemm_epilogue_rows(A: torch.Tensor, B: torch.Tensor, bias: Optional[torch.Tensor] = None, *,
                               gather: bool = False, compute=None, **kw) -> torch.Tensor:
    """Row-block (M) shard of one GEMM: rank r computes rows shard_range(M, r, P, 256) of C.
    A is the full (M, K) operand or the rank's row block (``presliced=True``, then a COL/FULL bias
    must be the rank's rows too); B and a ROW bias are replicated, a COL (M,) or FULL (M, ld) bias
    is sliced with A's rows."""
    from . import gemm_epilogue
    presliced = kw.pop("presliced", False)
    M = kw.pop("total_rows", A.shape[0])
    rank, world = _world()
    lo, hi = shard_range(M, rank, world, ROW_QUANTUM)
    if not presliced:
        A = A[lo:hi]
        if bias is not None and kw.get("bias_mode", "row") in ("col", "full"):
            bias = bias[lo:hi]          # bias[i] / bias[i, :] follow the rows of A
    fn = compute or gemm_epilogue
    C = fn(A, B, bias, **kw) if hi > lo else torch.empty((0, B.shape[1]), dtype=kw.get("out_dtype", torch.float16),
                                                         device=A.device)
    return gather_rows(C, M, ROW_QUANTUM) if gather else C
