"""Multi-process (world_size 2, gloo, CPU) tests of the sharding logic in
paper_2006_12645_b200/sharded.py.  The per-rank compute is the CPU oracle (tests may call it), so
these check the partitioning, slicing and gather, not the kernel (which is covered on the GPU)."""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import workloads
from paper_2006_12645_b200 import sharded


def test_shard_range_partitions():
    for n in (0, 1, 7, 64, 1000, 8192, 8193):
        for world in (1, 2, 3, 4, 8):
            for q in (1, 256):
                rs = sharded.all_ranges(n, world, q)
                assert rs[0][0] == 0 and rs[-1][1] == n
                for (a, b), (c, d) in zip(rs, rs[1:]):
                    assert b == c and a <= b
                for lo, hi in rs[:-1]:
                    assert lo % q == 0 and hi % q == 0 or hi == n
                sizes = [hi - lo for lo, hi in rs]
                if n >= q * world:
                    assert max(sizes) - min(sizes) < 2 * q     # balanced in whole quanta; ragged tail last


def _oracle_f16(A, B, bias, bias_mode="row", out_dtype=torch.float16, **_):
    M, K = A.shape
    N = B.shape[1]
    ldbias = bias.shape[-1] if (bias is not None and bias_mode == "full") else 0
    out, _ = oracle.gemm_epilogue(A.contiguous(), B.contiguous(), M, N, K, bias=bias, bias_mode=bias_mode,
                                  ldbias=ldbias, nthreads=2)
    if out_dtype == torch.float32:
        return torch.from_numpy(out.astype(np.float32))
    return torch.from_numpy(oracle.f16_encode(out).view(np.float16).copy())


def _oracle_batched(A, B, bias, bias_mode="row", out_dtype=torch.float16, **kw):
    per_item = bias is not None and bias.dim() == (3 if bias_mode == "full" else 2)
    items = [_oracle_f16(A[i], B[i], bias[i] if per_item else bias, bias_mode=bias_mode, out_dtype=out_dtype)
             for i in range(A.shape[0])]
    return torch.stack(items) if items else torch.empty((0, A.shape[1], B.shape[2]), dtype=out_dtype)


def _same(x, y):
    return x.dtype == y.dtype and x.shape == y.shape and torch.equal(x, y)


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        # batched: 5 items over 2 ranks (3 + 2), per-item bias, gathered everywhere
        probs = [workloads.make_problem(40, 24, 16, seed=600 + b, bias_mode="row") for b in range(5)]
        A = torch.stack([p.A for p in probs])
        B = torch.stack([p.B for p in probs])
        bias = torch.stack([p.bias for p in probs])
        lo, hi = sharded.shard_range(5, rank, world)
        local = sharded.sharded_gemm_epilogue_batched(A, B, bias, compute=_oracle_batched)
        assert local.shape[0] == hi - lo
        full = sharded.sharded_gemm_epilogue_batched(A, B, bias, gather=True, compute=_oracle_batched)
        ref = _oracle_batched(A, B, bias)
        ok_b = torch.equal(full.view(torch.int16), ref.view(torch.int16))
        # every bias shape of the batched path: shared (1-D / 2-D full) and per item (2-D / 3-D full)
        g = workloads.gen(610)
        bias_cases = {
            "row_shared": ("row", workloads.uniform_f16((24,), 611)),
            "col_item": ("col", workloads.uniform_f16((5, 40), 612)),
            "col_shared": ("col", workloads.uniform_f16((40,), 613)),
            "full_shared": ("full", workloads.uniform_f16((40, 32), 614)),
            "full_item": ("full", workloads.uniform_f16((5, 40, 24), 615)),
        }
        ok_bias = {}
        for name, (bm, bb) in bias_cases.items():
            got = sharded.sharded_gemm_epilogue_batched(A, B, bb, gather=True, compute=_oracle_batched, bias_mode=bm)
            ok_bias[name] = _same(got, _oracle_batched(A, B, bb, bias_mode=bm))
        # rows: M = 600 over 2 ranks, cut at 256-row multiples (512 + 88)
        p = workloads.make_problem(600, 40, 32, seed=700, bias_mode="row")
        full_r = sharded.sharded_gemm_epilogue_rows(p.A, p.B, p.bias, gather=True, compute=_oracle_f16)
        ok_r = torch.equal(full_r.view(torch.int16), _oracle_f16(p.A, p.B, p.bias).view(torch.int16))
        for name, bm, bb in (("rows_col", "col", workloads.uniform_f16((600,), 616)),
                             ("rows_full", "full", workloads.uniform_f16((600, 48), 617))):
            got = sharded.sharded_gemm_epilogue_rows(p.A, p.B, bb, gather=True, compute=_oracle_f16, bias_mode=bm)
            ok_bias[name] = _same(got, _oracle_f16(p.A, p.B, bb, bias_mode=bm))
        # fp32 output with a rank that owns nothing (1 item over 2 ranks; 200 rows < one 256-row block)
        one = sharded.sharded_gemm_epilogue_batched(A[:1], B[:1], bias[:1], gather=True, compute=_oracle_batched,
                                                    out_dtype=torch.float32)
        ok_bias["empty_rank_f32_batched"] = _same(one, _oracle_batched(A[:1], B[:1], bias[:1], out_dtype=torch.float32))
        pr = workloads.make_problem(200, 40, 32, seed=701, bias_mode="row")
        rr = sharded.sharded_gemm_epilogue_rows(pr.A, pr.B, pr.bias, gather=True, compute=_oracle_f16,
                                                out_dtype=torch.float32)
        ok_bias["empty_rank_f32_rows"] = _same(rr, _oracle_f16(pr.A, pr.B, pr.bias, out_dtype=torch.float32))
        lo_r, hi_r = sharded.shard_range(600, rank, world, sharded.ROW_QUANTUM)
        q.put((rank, ok_b, ok_r, (lo, hi), (lo_r, hi_r), ok_bias))
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def test_two_rank_gloo_shard_and_gather():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=240) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert [r[1] for r in res] == [True, True], "batched gather != single-process oracle"
    assert [r[2] for r in res] == [True, True], "row-sharded gather != single-process oracle"
    assert [r[3] for r in res] == [(0, 3), (3, 5)]
    assert [r[4] for r in res] == [(0, 512), (512, 600)]
    for r in res:
        assert all(r[5].values()), r[5]
