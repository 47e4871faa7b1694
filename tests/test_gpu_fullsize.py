"""GPU parity at BASELINE.json's full sizes, in the launch configuration bench.py uses (the
default tile heuristic).  Up to 4096^3 (<= 2^36 FMA) the WHOLE output matrix is
compared with the oracle in every layout; above that (8192^3, the batch) the check is sampled:
every element of the tile-boundary rows/columns {0, 127, 128, 255, 256, 511, 512, 1023, 1024,
last} (the 128-row CTA tile, the 256-row pair tile, the 512-column pair tile and their
neighbours) plus seeded random rows x columns (the oracle evaluates the cross product of the
sampled rows and columns).  Uniform data is held to the north_star bound and the ReLU invariant;
small-integer data (exact in fp32 in any order) bitwise."""
from __future__ import annotations

import functools

import numpy as np
import pytest
import torch

import oracle
import workloads
from tests.helpers import check_bound, check_relu_invariant, oracle_run

pytestmark = pytest.mark.gpu
ge = pytest.importorskip("paper_2006_12645_b200")


def sample_idx(n, k, seed):
    g = np.random.default_rng(seed)
    base = [i for i in (0, 127, 128, 255, 256, 511, 512, 1023, 1024, n - 1) if 0 <= i < n]
    extra = g.choice(n, size=min(k, n), replace=False)
    return np.unique(np.concatenate([base, extra])).astype(np.int64)


@functools.lru_cache(maxsize=2)
def problem(M, N, K, seed, kind, prologue=None):
    return workloads.make_problem(M, N, K, seed=seed, kind=kind, bias_mode="row", prologue=prologue)


def to_dev(prob, layouts, ldb=None, ldc=None):
    def put(logical, lay, ld):
        if ld is None:
            ld = (logical.shape[1 if lay == "r" else 0] + 7) // 8 * 8
        st, ld = workloads.store(logical, lay, ld)
        d = st.cuda()
        R, C = logical.shape
        return d[:, :C] if lay == "r" else d[:, :R].t()
    A = put(prob.A, layouts[0], None)
    B = put(prob.B, layouts[1], ldb)
    return A, B


def run_sampled(prob, layouts, rows, cols, ldb=None, ldc=None):
    A, B = to_dev(prob, layouts, ldb)
    if ldc is None:
        C = torch.empty((prob.M, prob.N), dtype=torch.float16, device="cuda")
    else:
        C = torch.empty((prob.M, ldc), dtype=torch.float16, device="cuda")[:, :prob.N]
    scale = prob.scale.cuda() if prob.scale is not None else None
    ge.gemm_epilogue(A, B, prob.bias.cuda(), prologue=prob.meta.get("prologue"), scale=scale, out=C)
    torch.cuda.synchronize()
    got = C[torch.as_tensor(rows, device="cuda")][:, torch.as_tensor(cols, device="cuda")]
    return got.float().cpu().numpy().astype(np.float64)


def check(prob, layouts, kind, nsamp=160, **kw):
    rows = sample_idx(prob.M, nsamp, 1)
    cols = sample_idx(prob.N, nsamp, 2)
    got = run_sampled(prob, layouts, rows, cols, **kw)
    pre, mag = oracle_run(prob, layouts, rows=rows, cols=cols, relu=False)
    out = np.where(pre > 0, pre, 0.0)          # relu(pre), pinned by test_relu_invariant (CPU)
    if kind == "smallint":
        assert np.array_equal(got, oracle.f16_decode(oracle.f16_encode(out))), layouts
    else:
        check_bound(got, out, mag, layouts)
        check_relu_invariant(got, pre, mag, layouts)


@pytest.mark.parametrize("kind", ["uniform", "smallint"])
@pytest.mark.parametrize("layouts", workloads.LAYOUTS)
def test_square_8192(layouts, kind):
    """BASELINE configs[1] at 8192^3 (the bench workload), all four layouts."""
    check(problem(8192, 8192, 8192, 51, kind), layouts, kind)


@functools.lru_cache(maxsize=1)
def full_oracle(n, seed, kind):
    """Full n x n oracle (pre-activation, mag) of the rr problem; the oracle is layout invariant
    bitwise (pinned on the CPU by test_layout_invariance_bitwise), so one evaluation serves all four
    layouts of the same logical operands."""
    return oracle_run(problem(n, n, n, seed, kind), "rr", relu=False)


def run_full(prob, layouts):
    A, B = to_dev(prob, layouts)
    C = torch.empty((prob.M, prob.N), dtype=torch.float16, device="cuda")
    ge.gemm_epilogue(A, B, prob.bias.cuda(), out=C)
    torch.cuda.synchronize()
    return C.float().cpu().numpy().astype(np.float64)


@pytest.mark.parametrize("n", [1024, 2048, 4096])
def test_square_full_matrix(n):
    """BASELINE configs[1] at 1024^3 / 2048^3 / 4096^3, all four layouts, EVERY output element against
    the oracle (north_star bound + ReLU invariant), in the bench's launch configuration."""
    prob = problem(n, n, n, 52, "uniform")
    pre, mag = full_oracle(n, 52, "uniform")
    out = np.where(pre > 0, pre, 0.0)
    for layouts in workloads.LAYOUTS:
        got = run_full(prob, layouts)
        check_bound(got, out, mag, f"{n}^3 {layouts}")
        nz, npos = check_relu_invariant(got, pre, mag, f"{n}^3 {layouts}")
        assert nz > n * n // 4 and npos > n * n // 4


def test_square_full_matrix_smallint_2048():
    """2048^3 small-integer data, all four layouts, the whole matrix bitwise equal to RNE(oracle)."""
    prob = problem(2048, 2048, 2048, 57, "smallint")
    pre, _ = full_oracle(2048, 57, "smallint")
    want = oracle.f16_decode(oracle.f16_encode(np.where(pre > 0, pre, 0.0)))
    for layouts in workloads.LAYOUTS:
        assert np.array_equal(run_full(prob, layouts), want), layouts


@pytest.mark.parametrize("kind", ["uniform", "smallint"])
@pytest.mark.parametrize("layouts", ["rr", "rc"])
def test_deepbench_5124x700x2048(layouts, kind):
    """BASELINE configs[2] (a): a wave-quantised rectangular shape, N not a tile multiple."""
    check(problem(5124, 700, 2048, 53, kind), layouts, kind)


@pytest.mark.parametrize("layouts", ["rr", "rc"])
def test_deepbench_35x8457x2560(layouts):
    """BASELINE configs[2] (b): skinny M=35, N=8457 with padded ldb/ldc (TMA path) and with the
    unpadded ldc=8457 (st.global epilogue)."""
    for kind in ("uniform", "smallint"):
        prob = problem(35, 8457, 2560, 54, kind)
        check(prob, layouts, kind, ldb=8464 if layouts[1] == "r" else None, ldc=8464)
        check(prob, layouts, kind, ldb=8464 if layouts[1] == "r" else None, ldc=8457)


@pytest.mark.parametrize("kind", ["uniform", "smallint"])
def test_prologue_4096(kind):
    """BASELINE configs[3]: SCALE_K prologue + bias + ReLU at 4096^3 (DESIGN.md R-C12)."""
    check(problem(4096, 4096, 4096, 55, kind, "scale_k"), "rr", kind)


def test_batched_64x2048():
    """BASELINE configs[4]: batch 64 x 2048^3 in one persistent launch, per-item bias; sampled
    items checked against the oracle, every item against the single-GEMM call (bitwise)."""
    batch, M, N, K = 64, 2048, 2048, 2048
    g = torch.Generator(device="cuda")
    g.manual_seed(56)
    A = (torch.rand(batch, M, K, generator=g, device="cuda") * 2 - 1).half()
    B = (torch.rand(batch, K, N, generator=g, device="cuda") * 2 - 1).half()
    bias = (torch.rand(batch, N, generator=g, device="cuda") * 2 - 1).half()
    C = ge.gemm_epilogue_batched(A, B, bias)
    from paper_2006_12645_b200 import sharded
    Cs = sharded.sharded_gemm_epilogue_batched(A, B, bias, total_batch=batch)   # bench's N > 1 path at world 1
    torch.cuda.synchronize()
    assert torch.equal(Cs, C)
    rows, cols = sample_idx(M, 64, 3), sample_idx(N, 64, 4)
    for b in (0, 17, 63):
        single = ge.gemm_epilogue(A[b], B[b], bias[b])
        torch.cuda.synchronize()
        assert torch.equal(single, C[b])
        out, mag = oracle.gemm_epilogue(A[b].cpu(), B[b].cpu(), M, N, K, bias=bias[b].cpu(), rows=rows, cols=cols)
        got = C[b].cpu()[torch.as_tensor(rows)][:, torch.as_tensor(cols)].float().numpy().astype(np.float64)
        check_bound(got, out, mag, f"item {b}")
