"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle, element by element.

Tolerance (BASELINE.json north_star): |gpu - oracle| <= 4e-3*mag + 1e-3*|oracle| per element,
mag = sum_k |a'_ik b_kj|.  Small-integer data is exact in fp32 in any summation order, so there
the GPU must equal RNE_fp16(oracle) (fp16 out) or the oracle itself (fp32 out) bitwise
(DESIGN.md "Parity").  All inputs are seeded (workloads.py)."""
from __future__ import annotations

import json
import os

import numpy as np
import pytest
import torch

import oracle
import workloads

from tests.helpers import check_bound, check_relu_invariant, oracle_run

pytestmark = pytest.mark.gpu

ge = pytest.importorskip("paper_2006_12645_b200")


def dev_operands(prob: workloads.Problem, layouts: str, lda=None, ldb=None):
    """Logical views on the GPU whose storage follows the layout pair (row/col major, padded ld)."""
    def put(logical, lay, ld):
        if ld is None:      # TMA needs 16-byte row pitch: pad the leading dimension to 8 elements
            ld = (logical.shape[1 if lay == "r" else 0] + 7) // 8 * 8
        st, ld = workloads.store(logical, lay, ld)
        d = st.cuda()
        R, C = logical.shape
        return d[:, :C] if lay == "r" else d[:, :R].t()
    return put(prob.A, layouts[0], lda), put(prob.B, layouts[1], ldb)


def dev_tile(logical, lay, ld=None):
    """A logical M x K tile on the GPU in layout `lay` (the Hadamard operand S follows A's layout)."""
    if ld is None:
        ld = (logical.shape[1 if lay == "r" else 0] + 7) // 8 * 8
    st, ld = workloads.store(logical, lay, ld)
    d = st.cuda()
    R, C = logical.shape
    return d[:, :C] if lay == "r" else d[:, :R].t()


def run_gpu(prob, layouts="rr", *, op=None, out_dtype=torch.float16, lda=None, ldb=None, **kw):
    A, B = dev_operands(prob, layouts, lda, ldb)
    bias = prob.bias.cuda() if prob.bias is not None else None
    scale = prob.scale.cuda() if prob.scale is not None else None
    if prob.meta.get("prologue") == "hadamard":
        scale = dev_tile(prob.scale, layouts[0])
    bm = prob.meta.get("bias_mode")
    C = ge.gemm_epilogue(A, B, bias, op=op, bias_mode=bm if bm in ("row", "col", "full") else "row",
                         prologue=prob.meta.get("prologue"), scale=scale, out_dtype=out_dtype, **kw)
    torch.cuda.synchronize()
    return C.float().cpu().numpy().astype(np.float64)


def exact_expect(out, out_dtype):
    return out if out_dtype == torch.float32 else oracle.f16_decode(oracle.f16_encode(out))


CONFIGS = [(64, 1), (128, 1), (192, 1), (256, 1), (128, 2), (192, 2), (256, 2), (512, 2)]


# ------------------------------------------------------------------ small full-matrix parity
@pytest.mark.parametrize("layouts", workloads.LAYOUTS)
@pytest.mark.parametrize("kind", ["uniform", "smallint"])
def test_layouts_ragged(layouts, kind):
    """All four layouts on a ragged 300x520x200 problem spanning several tiles."""
    prob = workloads.make_problem(300, 520, 200, seed=31, kind=kind, bias_mode="row")
    got = run_gpu(prob, layouts)
    pre, mag = oracle_run(prob, layouts, relu=False)
    out = np.where(pre > 0, pre, 0.0)          # relu(pre), pinned by test_relu_invariant (CPU)
    if kind == "smallint":
        assert np.array_equal(got, exact_expect(out, torch.float16))
    else:
        check_bound(got, out, mag, layouts)
        check_relu_invariant(got, pre, mag, layouts)


GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "hand_cases.json")


def _golden():
    with open(GOLDEN) as f:
        return json.load(f)["cases"]


@pytest.mark.parametrize("case", _golden(), ids=lambda c: c["name"])
@pytest.mark.parametrize("layouts", workloads.LAYOUTS)
def test_golden_cases_on_gpu(case, layouts):
    """The hand-computed cases of tests/golden/hand_cases.json (each citing its passage: Listing 1,
    Listing 5, the bias modes, the paper-literal rounding point R-C3, K = 0) through the CUDA path:
    every golden value is exactly computable in fp32, so the GPU must return RNE_fp16(golden)
    bitwise (fp16 out) and the golden value itself (fp32 out)."""
    M, N, K = case["M"], case["N"], case["K"]
    if K == 0 and layouts != "rr":
        pytest.skip("K = 0 is covered in rr (no operand is read)")
    A = torch.tensor(case["A"], dtype=torch.float16).reshape(M, K)
    B = torch.tensor(case["B"], dtype=torch.float16).reshape(K, N)
    bias = None if case["bias"] is None else torch.tensor(case["bias"], dtype=torch.float16)
    scale = None if case.get("scale") is None else torch.tensor(case["scale"], dtype=torch.float32)
    if case["prologue"] == "hadamard":
        scale = torch.tensor(case["S"], dtype=torch.float16).reshape(M, K)
    prob = workloads.Problem(M, N, K, A, B, bias, scale, {"bias_mode": case["bias_mode"], "prologue": case["prologue"]})
    op = ("bias_" if bias is not None else "") + ("relu" if case["relu"] else "")
    op = {"bias_": "bias", "": "none"}.get(op, op)
    if case.get("literal_round"):
        op = "literal_" + op
    want = np.array(case["out"], dtype=np.float64).reshape(M, N)
    for dt in (torch.float16, torch.float32):
        got = run_gpu(prob, layouts, op=op, out_dtype=dt)
        # fp32 out of the literal reading is the fp16-rounded pre-activation (exact in fp32)
        assert np.array_equal(got, exact_expect(want, dt)), (case["name"], layouts, dt, got, want)
        if case["relu"]:
            assert not np.signbit(got).any()


@pytest.mark.parametrize("tile_n,cg", CONFIGS)
@pytest.mark.parametrize("layouts", ["rc", "cr"])
def test_relu_invariant_uniform(tile_n, cg, layouts):
    """BASELINE.json north_star ReLU invariant on the GPU output for uniform data, every kernel
    configuration: C >= 0, no -0, exactly +0 where pre <= -tol and > 0 where pre >= tol."""
    if (tile_n, cg) == (192, 2) and layouts[1] == "r":
        pytest.skip("the 256 x 192 pair tile needs a K-major B")
    prob = workloads.make_problem(333, 777, 321, seed=30, kind="uniform", bias_mode="row")
    got = run_gpu(prob, layouts, tile_n=tile_n, cta_group=cg)
    pre, mag = oracle_run(prob, layouts, relu=False)
    nz, npos = check_relu_invariant(got, pre, mag, f"{tile_n}x{cg} {layouts}")
    assert nz > 1000 and npos > 1000
    check_bound(got, np.where(pre > 0, pre, 0.0), mag, "relu")


@pytest.mark.parametrize("tile_n,cg", CONFIGS)
@pytest.mark.parametrize("layouts", workloads.LAYOUTS)
def test_tile_configs_exact(tile_n, cg, layouts):
    """Every kernel configuration (N tile 64/128/256, 1-CTA and CTA-pair) is bitwise exact on
    small-integer data, with M/N/K tails (M=333, N=777, K=321)."""
    prob = workloads.make_problem(333, 777, 321, seed=32, kind="smallint", bias_mode="row")
    if (tile_n, cg) == (192, 2) and layouts[1] == "r":
        with pytest.raises(ge.GEError):            # the 256 x 192 pair tile needs a K-major B
            run_gpu(prob, layouts, tile_n=tile_n, cta_group=cg)
        return
    got = run_gpu(prob, layouts, tile_n=tile_n, cta_group=cg)
    out, _ = oracle_run(prob, layouts)
    assert np.array_equal(got, exact_expect(out, torch.float16))


@pytest.mark.parametrize("bias_mode", ["row", "col", "full"])
@pytest.mark.parametrize("out_dtype", [torch.float16, torch.float32])
@pytest.mark.parametrize("op", ["none", "bias", "relu", "bias_relu"])
def test_epilogue_variants(bias_mode, out_dtype, op):
    """Bias modes (DESIGN.md R-C2), epilogue ops and fp16/fp32 outputs, exact on small integers."""
    prob = workloads.make_problem(200, 300, 130, seed=33, kind="smallint", bias_mode=bias_mode,
                                  ldbias=312 if bias_mode == "full" else None)
    got = run_gpu(prob, "rc", op=op, out_dtype=out_dtype)
    use_bias = op in ("bias", "bias_relu")
    out, _ = oracle_run(prob, "rc", relu=op in ("relu", "bias_relu"), bias_mode=bias_mode if use_bias else "none")
    assert np.array_equal(got, exact_expect(out, out_dtype))


@pytest.mark.parametrize("prologue", ["scale_k", "relu", "hadamard"])
@pytest.mark.parametrize("layouts", workloads.LAYOUTS)
@pytest.mark.parametrize("tile_n,cg", [(256, 1), (256, 2), (64, 1), (512, 2), (128, 2), (192, 1)])
def test_prologue(prologue, layouts, tile_n, cg):
    """Prologue fusion (Sec. VII-C; SCALE_K = DESIGN.md R-C12, HADAMARD = R-C18,
    the full-tile op with a second input dataspace): the transform warps load A
    (and S) from global memory, apply the op in registers and store the swizzled stage; exact on
    small integers (s in {0.5, 1, 2}; S in {-1, 0.5, 1, 2}), within the bound on uniform data, with
    M/N/K tails (257 x 300 x 200: a partial last row tile and a K tail inside one 16-B chunk)."""
    for kind in ("smallint", "uniform"):
        prob = workloads.make_problem(257, 300, 200, seed=34, kind=kind, bias_mode="row", prologue=prologue)
        got = run_gpu(prob, layouts, tile_n=tile_n, cta_group=cg)
        out, mag = oracle_run(prob, layouts)
        if kind == "smallint":
            assert np.array_equal(got, exact_expect(out, torch.float16))
        else:
            check_bound(got, out, mag, f"{prologue} {layouts}")


@pytest.mark.parametrize("prologue", ["scale_k", "relu"])
@pytest.mark.parametrize("layouts", ["rr", "cc"])
def test_prologue_multi_tile(prologue, layouts):
    """The in-place prologue transform over several tiles per CTA pair (100 tiles of 256 x 256 on at
    most 74 pairs) and 16 k-blocks, so every ring slot is transformed many times across tiles:
    bitwise equal to the 256 x 512 tile's launch on small integers (exact in any order), fp16 and
    fp32 out, and within the bound of the oracle on a sample of rows/columns of uniform data."""
    M, N, K = 2560, 2560, 1024
    prob = workloads.make_problem(M, N, K, seed=77, kind="smallint", bias_mode="row", prologue=prologue)
    for dt in (torch.float16, torch.float32):
        ta = run_gpu(prob, layouts, tile_n=256, cta_group=2, out_dtype=dt)
        ref = run_gpu(prob, layouts, tile_n=512, cta_group=2, out_dtype=dt)
        assert np.array_equal(ta, ref), (prologue, layouts, dt)
    prob = workloads.make_problem(M, N, K, seed=78, kind="uniform", bias_mode="row", prologue=prologue)
    got = run_gpu(prob, layouts, tile_n=256, cta_group=2)
    rows, cols = np.array([0, 127, 128, 255, 256, 1300, M - 1]), np.array([0, 63, 64, 127, 128, 255, 256, 1111, N - 1])
    out, mag = oracle_run(prob, layouts, rows=rows, cols=cols)
    check_bound(got[np.ix_(rows, cols)], out, mag, f"multi-tile {prologue} {layouts}")


@pytest.mark.parametrize("M,N,K", [(1, 1, 1), (8, 8, 8), (1, 300, 64), (300, 1, 64), (127, 129, 63), (128, 256, 64),
                                   (129, 257, 65), (64, 64, 4096), (1000, 72, 17)])
def test_odd_shapes(M, N, K):
    prob = workloads.make_problem(M, N, K, seed=35, kind="smallint", bias_mode="row")
    for lay in ("rr", "cc"):
        got = run_gpu(prob, lay)
        out, _ = oracle_run(prob, lay)
        assert np.array_equal(got, exact_expect(out, torch.float16)), lay


def test_k_zero_and_empty():
    """K = 0 gives op(bias) (DESIGN.md R-C9); M = 0 / N = 0 are no-ops."""
    prob = workloads.make_problem(70, 90, 0, seed=36, bias_mode="col")
    got = run_gpu(prob, "rr")
    b = prob.bias.float().numpy().astype(np.float64)[:, None] + np.zeros((70, 90))
    assert np.array_equal(got, np.where(b > 0, b, 0.0))
    A = torch.zeros((0, 64), dtype=torch.float16, device="cuda")
    B = torch.zeros((64, 32), dtype=torch.float16, device="cuda")
    assert ge.gemm_epilogue(A, B).shape == (0, 32)


def test_padded_ld_and_c_fallback():
    """Padded lda/ldb; a C whose ldc breaks the 16-byte TMA rule goes through the st.global epilogue
    (the DeepBench N = 8457 case)."""
    prob = workloads.make_problem(150, 37, 100, seed=37, kind="smallint", bias_mode="row")
    A, B = dev_operands(prob, "cr", lda=160, ldb=40)
    Cbuf = torch.full((150, 37), 7.0, dtype=torch.float16, device="cuda")       # ldc = 37: misaligned rows
    ge.gemm_epilogue(A, B, prob.bias.cuda(), out=Cbuf)
    torch.cuda.synchronize()
    out, _ = oracle_run(prob, "cr")
    assert np.array_equal(Cbuf.float().cpu().numpy(), exact_expect(out, torch.float16))
    # misaligned base pointer of C (offset by one element) and fp32 output
    big = torch.zeros(150 * 40 + 1, dtype=torch.float32, device="cuda")
    Cv = big[1:].view(150, 40)[:, :37]
    ge.gemm_epilogue(A, B, prob.bias.cuda(), out=Cv)
    torch.cuda.synchronize()
    assert np.array_equal(Cv.cpu().numpy().astype(np.float64), out)


def test_padding_untouched():
    """Only the M x N window of C is written (ldc > N, the padding keeps its contents)."""
    prob = workloads.make_problem(130, 200, 64, seed=38, kind="smallint", bias_mode="row")
    A, B = dev_operands(prob, "rr")
    Cbuf = torch.full((130, 256), -5.0, dtype=torch.float16, device="cuda")
    ge.gemm_epilogue(A, B, prob.bias.cuda(), out=Cbuf[:, :200])
    torch.cuda.synchronize()
    assert (Cbuf[:, 200:] == -5.0).all()


@pytest.mark.parametrize("out_dtype", [torch.float16, torch.float32])
@pytest.mark.parametrize("M,N,swap", [(64, 1030, 1), (300, 1027, 1), (35, 1030, 2), (35, 1027, 2), (300, 701, 1)])
def test_padding_untouched_ragged_width(M, N, swap, out_dtype):
    """A C width that is not a multiple of 16 B with a padded ldc (16-B aligned rows, so the TMA store
    path): the TMA store clips its inner dimension only at 16-B granularity, so the library maps C's
    width rounded down and writes the ragged edge element-wise; the padding past column N keeps its
    contents and every element of C is right (bitwise, small integers), swapped and unswapped, batched."""
    batch, K = 2, 136
    probs = [workloads.make_problem(M, N, K, seed=150 + b, kind="smallint", bias_mode="row") for b in range(batch)]
    A = torch.stack([p.A for p in probs]).cuda()
    ldb = (N + 7) // 8 * 8
    Bpad = torch.zeros((batch, K, ldb), dtype=torch.float16)
    Bpad[:, :, :N] = torch.stack([p.B for p in probs])
    B = Bpad.cuda()[:, :, :N]
    bias = torch.stack([p.bias for p in probs]).cuda()
    Cbuf = torch.full((batch, M, 1040), -5.0, dtype=out_dtype, device="cuda")
    ge.gemm_epilogue_batched(A, B, bias, out=Cbuf[:, :, :N], swap_ab=swap)
    torch.cuda.synchronize()
    assert (Cbuf[:, :, N:] == -5.0).all()
    for b, p in enumerate(probs):
        out, _ = oracle_run(p, "rr")
        assert np.array_equal(Cbuf[b, :, :N].float().cpu().numpy().astype(np.float64), exact_expect(out, out_dtype))


@pytest.mark.parametrize("shared_bias", [True, False])
def test_batched_matches_single(shared_bias):
    """Item b of the batched call equals the single call on item b, bitwise (DESIGN.md R-C14)."""
    batch, M, N, K = 5, 200, 136, 96
    probs = [workloads.make_problem(M, N, K, seed=400 + b, bias_mode="row") for b in range(batch)]
    A = torch.stack([p.A for p in probs]).cuda()
    B = torch.stack([p.B for p in probs]).cuda().transpose(1, 2).contiguous().transpose(1, 2)  # col-major items
    bias = probs[0].bias.cuda() if shared_bias else torch.stack([p.bias for p in probs]).cuda()
    C = ge.gemm_epilogue_batched(A, B, bias)
    for b in range(batch):
        Cb = ge.gemm_epilogue(A[b], B[b], bias if shared_bias else bias[b])
        torch.cuda.synchronize()
        assert torch.equal(C[b], Cb)
        p = probs[b]
        if shared_bias:
            p = workloads.Problem(M, N, K, p.A, p.B, probs[0].bias, None, p.meta)
        out, mag = oracle_run(p, "rc")
        check_bound(C[b].float().cpu().numpy(), out, mag, f"item {b}")


def test_deterministic():
    prob = workloads.make_problem(512, 512, 512, seed=39, bias_mode="row")
    A, B = dev_operands(prob, "rr")
    bias = prob.bias.cuda()
    c1 = ge.gemm_epilogue(A, B, bias)
    c2 = ge.gemm_epilogue(A, B, bias)
    torch.cuda.synchronize()
    assert torch.equal(c1, c2)


def test_errors_raise():
    A = torch.zeros((64, 64), dtype=torch.float16, device="cuda")
    B = torch.zeros((64, 64), dtype=torch.float16, device="cuda")
    buf = torch.zeros(64 * 64 + 1, dtype=torch.float16, device="cuda")
    with pytest.raises(ge.GEError) as e:
        ge.gemm_epilogue(buf[1:].view(64, 64), B)                  # 2-byte offset base: TMA needs 16 B
    assert e.value.status == ge.Status.MISALIGNED
    with pytest.raises(ge.GEError) as e:
        ge.gemm_epilogue(A, B, out=A)                              # C aliases A
    assert e.value.status == ge.Status.ALIASING


def test_host_entry_point():
    """gemm_epilogue_host (host buffers, copies inside the call) equals the device-pointer path."""
    prob = workloads.make_problem(300, 264, 200, seed=40, bias_mode="row")
    Ah = prob.A.pin_memory()
    Bh = prob.B.t().contiguous().pin_memory().t()
    Ch = ge.gemm_epilogue_host(Ah, Bh, prob.bias.pin_memory())
    Cd = ge.gemm_epilogue(Ah.cuda(), Bh.t().contiguous().cuda().t(), prob.bias.cuda())
    torch.cuda.synchronize()
    assert torch.equal(Ch, Cd.cpu())


# ------------------------------------------------------------------ stream-K
@pytest.mark.parametrize("M,N,K,tile_n,cg", [(1024, 1024, 1024, 256, 2), (640, 3000, 960, 256, 2),
                                            (2048, 768, 4096, 256, 1), (300, 520, 200, 128, 1),
                                            (4096, 4096, 256, 256, 2), (512, 512, 128, 64, 1)])
@pytest.mark.parametrize("layouts", ["rr", "cc"])
def test_stream_k_exact_and_bound(M, N, K, tile_n, cg, layouts):
    """Stream-K split of the last wave: bias+ReLU applied once after the full reduction (R-C13);
    small integers stay bitwise exact, uniform data within the bound."""
    p = ge.plan(M, N, K, tile_n=tile_n, cta_group=cg, stream_k=2)
    assert p["stream_k_tiles"] > 0
    for kind in ("smallint", "uniform"):
        prob = workloads.make_problem(M, N, K, seed=41, kind=kind, bias_mode="row")
        got = run_gpu(prob, layouts, tile_n=tile_n, cta_group=cg, stream_k=2)
        out, mag = oracle_run(prob, layouts)
        if kind == "smallint":
            assert np.array_equal(got, exact_expect(out, torch.float16))
        else:
            check_bound(got, out, mag, f"stream-K {M}x{N}x{K}")


def test_stream_k_deterministic_repeated_and_graph():
    """Fixed-order partial reduction: bitwise reproducible across launches, across a CUDA graph
    replay, and equal to the data-parallel result within the bound; flags are left reset."""
    prob = workloads.make_problem(2048, 2048, 2048, seed=42, bias_mode="col")
    A, B = dev_operands(prob, "rc")
    bias = prob.bias.cuda()
    kw = dict(bias_mode="col", tile_n=256, cta_group=2, stream_k=2)
    cs = torch.cuda.Stream()          # the workspace is per (device, stream) and never allocated
    with torch.cuda.stream(cs):       # while capturing: create it with an eager launch first
        c1 = ge.gemm_epilogue(A, B, bias, **kw)
        c2 = ge.gemm_epilogue(A, B, bias, **kw)
    cs.synchronize()
    out = torch.empty_like(c1)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=cs):
        ge.gemm_epilogue(A, B, bias, out=out, **kw)
    for _ in range(3):
        out.zero_()
        g.replay()
        torch.cuda.synchronize()
        assert torch.equal(out, c1)
    torch.cuda.synchronize()
    assert torch.equal(c1, c2)
    dp = ge.gemm_epilogue(A, B, bias, bias_mode="col", tile_n=256, cta_group=2, stream_k=1)
    torch.cuda.synchronize()
    o, m = oracle_run(prob, "rc")
    check_bound(c1.float().cpu().numpy(), o, m, "stream-K")
    check_bound(dp.float().cpu().numpy(), o, m, "data-parallel")


def test_stream_k_library_workspace_via_host_entry():
    """The host-buffer entry passes no workspace: the library-managed per-device buffer is used."""
    prob = workloads.make_problem(1024, 1024, 1024, seed=43, kind="smallint", bias_mode="row")
    Ch = ge.gemm_epilogue_host(prob.A, prob.B, prob.bias, tile_n=256, cta_group=2, stream_k=2)
    out, _ = oracle_run(prob, "rr")
    assert np.array_equal(Ch.float().numpy().astype(np.float64), exact_expect(out, torch.float16))


# ------------------------------------------------------------------ split-K (few, long tiles)
SPLIT_SHAPES = [(640, 1024, 3840), (2048, 128, 3456), (128, 2176, 3200), (384, 768, 1536), (300, 520, 2000)]


@pytest.mark.parametrize("M,N,K", SPLIT_SHAPES)
@pytest.mark.parametrize("layouts", workloads.LAYOUTS)
def test_split_k_exact_and_bound(M, N, K, layouts):
    """Split-K reduce-scatter: bias and activation applied once, after the full
    reduction (R-C13); bitwise exact on small integers, within the bound on uniform data."""
    p = ge.plan(M, N, K, layouts=layouts)
    assert p["split_k"] > 1, p
    for kind in ("smallint", "uniform"):
        prob = workloads.make_problem(M, N, K, seed=45, kind=kind, bias_mode="row")
        got = run_gpu(prob, layouts)
        out, mag = oracle_run(prob, layouts)
        if kind == "smallint":
            assert np.array_equal(got, exact_expect(out, torch.float16))
        else:
            check_bound(got, out, mag, f"split-K {M}x{N}x{K} {layouts}")


def test_split_k_deterministic_and_graph():
    """Fixed-order DSMEM reduction: bitwise reproducible across launches and CUDA-graph replays,
    equal to the data-parallel result within the bound."""
    M, N, K = 640, 1024, 3840
    assert ge.plan(M, N, K, layouts="rc")["split_k"] > 1
    prob = workloads.make_problem(M, N, K, seed=46, bias_mode="row")
    A, B = dev_operands(prob, "rc")
    bias = prob.bias.cuda()
    c1 = ge.gemm_epilogue(A, B, bias)
    c2 = ge.gemm_epilogue(A, B, bias)
    out = torch.empty_like(c1)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        ge.gemm_epilogue(A, B, bias, out=out)
    for _ in range(3):
        out.zero_()
        g.replay()
        torch.cuda.synchronize()
        assert torch.equal(out, c1)
    assert torch.equal(c1, c2)
    dp = ge.gemm_epilogue(A, B, bias, stream_k=1)
    torch.cuda.synchronize()
    o, m = oracle_run(prob, "rc")
    check_bound(c1.float().cpu().numpy(), o, m, "split-K")
    check_bound(dp.float().cpu().numpy(), o, m, "data-parallel")


@pytest.mark.parametrize("variant", ["f32_out", "col_bias", "prologue", "batched", "gemm2", "sigmoid"])
def test_split_k_variants(variant):
    """Split-K composes with fp32 output, COL bias, the prologue transform, batching, the sum of
    matmuls and a non-ReLU root op (exact on small integers / within the bound)."""
    M, N, K = 384, 640, 3072
    if variant == "prologue":
        prob = workloads.make_problem(M, N, K, seed=47, kind="smallint", bias_mode="row", prologue="scale_k")
        assert ge.plan(M, N, K, layouts="rc", prologue="scale_k")["split_k"] > 1
        got = run_gpu(prob, "rc")
        out, _ = oracle_run(prob, "rc")
        assert np.array_equal(got, exact_expect(out, torch.float16))
    elif variant in ("f32_out", "col_bias", "sigmoid"):
        bm = "col" if variant == "col_bias" else "row"
        kind = "uniform" if variant == "sigmoid" else "smallint"
        prob = workloads.make_problem(M, N, K, seed=48, kind=kind, bias_mode=bm)
        dt = torch.float32 if variant == "f32_out" else torch.float16
        op = "bias_sigmoid" if variant == "sigmoid" else None
        got = run_gpu(prob, "rc", out_dtype=dt, op=op)
        out, mag = oracle_run(prob, "rc", act="sigmoid" if variant == "sigmoid" else "default")
        if variant == "sigmoid":
            check_bound(got, out, mag, "split-K sigmoid")
        else:
            assert np.array_equal(got, exact_expect(out, dt))
    elif variant == "batched":
        batch = 3
        assert ge.plan(M, N, K, batch=batch, layouts="rr")["split_k"] > 1
        probs = [workloads.make_problem(M, N, K, seed=49 + i, kind="smallint", bias_mode="row") for i in range(batch)]
        A = torch.stack([q.A for q in probs]).cuda()
        B = torch.stack([q.B for q in probs]).cuda()
        bias = torch.stack([q.bias for q in probs]).cuda()
        C = ge.gemm_epilogue_batched(A, B, bias)
        torch.cuda.synchronize()
        for i, q in enumerate(probs):
            out, _ = oracle_run(q, "rr")
            assert np.array_equal(C[i].float().cpu().numpy().astype(np.float64), exact_expect(out, torch.float16))
    else:
        K1, K2 = 1536, 1536
        p1 = workloads.make_problem(M, N, K1, seed=52, kind="smallint", bias_mode="row")
        p2 = workloads.make_problem(M, N, K2, seed=53, kind="smallint", bias_mode="row")
        C = ge.gemm2_epilogue(p1.A.cuda(), p1.B.cuda(), p2.A.cuda(), p2.B.cuda(), p1.bias.cuda())
        torch.cuda.synchronize()
        out, _ = oracle.gemm2_epilogue(p1.A, p1.B, p2.A, p2.B, M, N, K1, K2, bias=p1.bias, bias_mode="row")
        assert np.array_equal(C.float().cpu().numpy().astype(np.float64), exact_expect(out, torch.float16))


# ------------------------------------------------------------------ the paper's pointwise op set
OPS = {"sigmoid": (None, False), "bias_sigmoid": ("sigmoid", False), "tanh": (None, False),
       "bias_tanh": ("tanh", False), "sub_bias": (None, True), "sub_bias_relu": ("relu", True),
       "sub_bias_sigmoid": ("sigmoid", True), "sub_bias_tanh": ("tanh", True)}


@pytest.mark.parametrize("op", sorted(OPS))
@pytest.mark.parametrize("tile_n,cg", [(512, 2), (256, 2), (64, 1)])
def test_pointwise_ops(op, tile_n, cg):
    """add / subtract bias then ReLU / Sigmoid / Tanh at the root,
    within the north_star bound (sigmoid' <= 1/4 and tanh' <= 1 do not amplify the pre-activation
    error); bias-subtracting identity ops stay bitwise exact on small integers."""
    act = "sigmoid" if "sigmoid" in op else "tanh" if "tanh" in op else "relu" if "relu" in op else None
    use_bias = "bias" in op
    sub = op.startswith("sub")
    for kind in ("uniform", "smallint"):
        prob = workloads.make_problem(300, 520, 200, seed=44, kind=kind, bias_mode="row")
        if not use_bias:
            prob = workloads.Problem(prob.M, prob.N, prob.K, prob.A, prob.B, None, None,
                                     {"bias_mode": None, "prologue": None})
        got = run_gpu(prob, "rc", op=op, tile_n=tile_n, cta_group=cg)
        out, mag = oracle_run(prob, "rc", act=act, bias_sub=sub)
        if kind == "smallint" and act in (None, "relu"):
            assert np.array_equal(got, exact_expect(out, torch.float16)), op
        else:
            check_bound(got, out, mag, op)


# ------------------------------------------------------------------ sum of matmuls (Listing 4)
@pytest.mark.parametrize("layouts", workloads.LAYOUTS)
@pytest.mark.parametrize("tile_n,cg", [(512, 2), (256, 2), (128, 1)])
def test_gemm2_sum_of_matmuls(layouts, tile_n, cg):
    """Z = relu(A.B + P.Q + bias) in one kernel, K1 != K2 with K tails:
    bitwise exact on small integers, within the bound on uniform data."""
    M, N, K1, K2 = 300, 520, 200, 136
    for kind in ("smallint", "uniform"):
        p1 = workloads.make_problem(M, N, K1, seed=45, kind=kind, bias_mode="row")
        p2 = workloads.make_problem(M, N, K2, seed=46, kind=kind, bias_mode=None)
        A, B = dev_operands(p1, layouts)
        P, Q = dev_operands(p2, layouts)
        C = ge.gemm2_epilogue(A, B, P, Q, p1.bias.cuda(), tile_n=tile_n, cta_group=cg)
        torch.cuda.synchronize()
        got = C.float().cpu().numpy().astype(np.float64)
        out, mag = oracle.gemm2_epilogue(p1.A, p1.B, p2.A, p2.B, M, N, K1, K2, bias=p1.bias, act="relu")
        if kind == "smallint":
            assert np.array_equal(got, exact_expect(out, torch.float16))
        else:
            check_bound(got, out, mag, "gemm2")


@pytest.mark.parametrize("layouts,bias_mode", [("rr", "col"), ("cr", "full"), ("cc", "row")])
def test_host_entry_pipelined_blocks(layouts, bias_mode):
    """The pipelined host path (row blocks of A/C streamed on copy/compute streams) equals the
    device path bitwise, for row- and column-major A and every bias mode; M spans 3 blocks."""
    M, N, K = 2304 + 40, 264, 136
    prob = workloads.make_problem(M, N, K, seed=47, bias_mode=bias_mode, ldbias=272 if bias_mode == "full" else None)
    def host_view(logical, lay):
        st, ld = workloads.store(logical, lay, (logical.shape[1 if lay == "r" else 0] + 7) // 8 * 8)
        st = st.pin_memory()
        R, Cc = logical.shape
        return st[:, :Cc] if lay == "r" else st[:, :R].t()
    Ah, Bh = host_view(prob.A, layouts[0]), host_view(prob.B, layouts[1])
    bh = prob.bias.pin_memory()
    kw = dict(bias_mode=bias_mode, tile_n=256, cta_group=2, stream_k=1)
    Ch = ge.gemm_epilogue_host(Ah, Bh, bh, **kw)
    A, B = dev_operands(prob, layouts)
    Cd = ge.gemm_epilogue(A, B, prob.bias.cuda(), **kw)
    torch.cuda.synchronize()
    assert torch.equal(Ch, Cd.cpu())


def test_host_entry_batched_items():
    batch, M, N, K = 5, 256, 192, 128
    probs = [workloads.make_problem(M, N, K, seed=500 + b, bias_mode="row") for b in range(batch)]
    A = torch.stack([p.A for p in probs]).pin_memory()
    B = torch.stack([p.B for p in probs]).pin_memory()
    bias = torch.stack([p.bias for p in probs]).pin_memory()
    kw = dict(tile_n=128, cta_group=1, stream_k=1)     # same kernel configuration on both paths
    Ch = ge.gemm_epilogue_host(A, B, bias, **kw)
    Cd = ge.gemm_epilogue_batched(A.cuda(), B.cuda(), bias.cuda(), **kw)
    torch.cuda.synchronize()
    assert torch.equal(Ch, Cd.cpu())


# ------------------------------------------------------------------ paper-literal rounding point (R-C3)
def _eighths_problem(M, N, K, seed):
    """a = u/64, bias = v/64 (u, v ~ U{-255..255}), b ~ U{-3..3}: every product and partial sum is
    exact in fp32 (<= 17 significant bits) but generally NOT representable in fp16, so the
    paper-literal fp16 rounding of the accumulator changes results while
    staying exactly computable on both sides."""
    g = torch.Generator().manual_seed(seed)
    A = (torch.randint(-255, 256, (M, K), generator=g).double() / 64).half()
    B = torch.randint(-3, 4, (K, N), generator=g).half()
    bias = (torch.randint(-255, 256, (N,), generator=g).double() / 64).half()
    return workloads.Problem(M, N, K, A, B, bias, None, {"bias_mode": "row", "prologue": None})


@pytest.mark.parametrize("tile_n,cg", [(512, 2), (256, 2), (128, 1)])
@pytest.mark.parametrize("out_dtype", [torch.float16, torch.float32])
def test_literal_rounding_point(tile_n, cg, out_dtype):
    """GE_EPI_F16_INTERMEDIATE: relu(fp16(fp16(acc) + bias)) (DESIGN.md R-C3).  On data whose fp32
    accumulation is exact the GPU equals the oracle's literal reading bitwise, and the flag is
    observable (it differs from the default single-rounding result somewhere); on uniform data
    both readings stay within the north_star bound."""
    prob = _eighths_problem(300, 520, 96, seed=61)
    got = run_gpu(prob, "rr", op="literal_bias_relu", out_dtype=out_dtype, tile_n=tile_n, cta_group=cg)
    lit, _ = oracle_run(prob, "rr", literal_round=True)
    assert np.array_equal(got, exact_expect(lit, out_dtype))
    default = run_gpu(prob, "rr", op="bias_relu", out_dtype=out_dtype, tile_n=tile_n, cta_group=cg)
    assert not np.array_equal(got, default)
    uni = workloads.make_problem(200, 300, 700, seed=62, kind="uniform", bias_mode="row")
    got_u = run_gpu(uni, "rc", op="literal_bias_relu", out_dtype=out_dtype, tile_n=tile_n, cta_group=cg)
    out, mag = oracle_run(uni, "rc")
    check_bound(got_u, out, mag, "literal vs exact")


def test_literal_rounding_split_k_and_no_bias():
    """The literal rounding happens once, after the full K reduction (split-K shapes), and with no
    bias it reduces to act(fp16(acc))."""
    prob = _eighths_problem(128, 256, 64 * 40, seed=63)
    got = run_gpu(prob, "rr", op="literal_bias_relu")
    lit, _ = oracle_run(prob, "rr", literal_round=True)
    assert np.array_equal(got, exact_expect(lit, torch.float16))
    nob = workloads.Problem(prob.M, prob.N, prob.K, prob.A, prob.B, None, None, {"bias_mode": None, "prologue": None})
    got = run_gpu(nob, "rr", op="literal_relu", out_dtype=torch.float32)
    lit, _ = oracle_run(nob, "rr", literal_round=True)
    assert np.array_equal(got, lit)


# ------------------------------------------------------------------ multicast clusters of two CTA pairs
@pytest.mark.parametrize("tile_n", [512, 256])
@pytest.mark.parametrize("layouts", workloads.LAYOUTS)
def test_multicast_clusters_exact(tile_n, layouts):
    """Clusters of two CTA pairs sharing B by TMA multicast (512 x tile_n tiles): bitwise exact on
    small integers and within the bound on uniform data, with a ragged M whose last cluster tile
    leaves the second pair entirely out of range (rows 768.. of M = 700) and ragged N, K."""
    for kind in ("smallint", "uniform"):
        prob = workloads.make_problem(700, 600, 200, seed=71, kind=kind, bias_mode="row")
        got = run_gpu(prob, layouts, tile_n=tile_n, cta_group=2, multicast=2)
        out, mag = oracle_run(prob, layouts)
        if kind == "smallint":
            assert np.array_equal(got, exact_expect(out, torch.float16))
        else:
            check_bound(got, out, mag, f"mc {tile_n} {layouts}")


@pytest.mark.parametrize("variant", ["f32_col", "full_bias", "batched", "gemm2", "long_k"])
def test_multicast_variants(variant):
    """fp32 output with a column bias, a full M x N bias, strided batches, the sum of matmuls and a
    long K (many ring wraps) through the multicast configuration, bitwise exact on small integers."""
    if variant == "batched":
        probs = [workloads.make_problem(600, 520, 136, seed=80 + b, kind="smallint", bias_mode="row") for b in range(3)]
        A = torch.stack([p.A for p in probs]).cuda()
        B = torch.stack([p.B for p in probs]).cuda()
        bias = torch.stack([p.bias for p in probs]).cuda()
        C = ge.gemm_epilogue_batched(A, B, bias, tile_n=512, cta_group=2, multicast=2)
        torch.cuda.synchronize()
        for b, p in enumerate(probs):
            out, _ = oracle_run(p, "rr")
            assert np.array_equal(C[b].float().cpu().numpy().astype(np.float64), exact_expect(out, torch.float16))
        return
    if variant == "gemm2":
        p1 = workloads.make_problem(1100, 700, 96, seed=90, kind="smallint", bias_mode="row")
        p2 = workloads.make_problem(1100, 700, 160, seed=91, kind="smallint", bias_mode="row")
        C = ge.gemm2_epilogue(p1.A.cuda(), p1.B.t().contiguous().t().cuda(), p2.A.cuda(),
                              p2.B.t().contiguous().t().cuda(), p1.bias.cuda(), tile_n=256, cta_group=2, multicast=2)
        torch.cuda.synchronize()
        out, _ = oracle.gemm2_epilogue(p1.A, p1.B, p2.A, p2.B, 1100, 700, 96, 160, bias=p1.bias, bias_mode="row")
        assert np.array_equal(C.float().cpu().numpy().astype(np.float64), exact_expect(out, torch.float16))
        return
    if variant == "long_k":
        prob = workloads.make_problem(1024, 512, 64 * 37 + 5, seed=92, kind="smallint", bias_mode="row")
        got = run_gpu(prob, "cr", tile_n=512, cta_group=2, multicast=2)
        out, _ = oracle_run(prob, "cr")
        assert np.array_equal(got, exact_expect(out, torch.float16))
        return
    bias_mode = "col" if variant == "f32_col" else "full"
    dt = torch.float32 if variant == "f32_col" else torch.float16
    prob = workloads.make_problem(900, 530, 150, seed=93, kind="smallint", bias_mode=bias_mode)
    got = run_gpu(prob, "rc", out_dtype=dt, tile_n=512, cta_group=2, multicast=2)
    out, _ = oracle_run(prob, "rc")
    assert np.array_equal(got, exact_expect(out, dt))


def test_multicast_rejects_prologue():
    prob = workloads.make_problem(600, 512, 128, seed=94, kind="smallint", bias_mode="row", prologue="scale_k")
    with pytest.raises(ge.GEError):
        run_gpu(prob, "rr", multicast=2)


@pytest.mark.parametrize("tile_n,cg", CONFIGS)
@pytest.mark.parametrize("out_dtype", [torch.float16, torch.float32])
@pytest.mark.parametrize("N", [1096, 1100])       # TMA store / st.global fallback (row pitch not 16-B aligned)
def test_fast_epilogue_matches_general(tile_n, cg, out_dtype, N):
    """The straight-line epilogue of the measured configuration (ROW bias + ReLU: FADD2, max(v,+0),
    one RNE pack) against the general epilogue code on the same accumulators: FULL bias holding
    the row bias broadcast to every row takes the general path and must agree bitwise (same fp32
    add, same ReLU, same rounding; DESIGN.md R-C5/R-C6).  Uniform data (no exactness needed: both
    read one accumulator), several 32-column chunks per warp, a ragged tail, zero rows in A (ReLU
    of +-0 bias: no -0 may reach C), and the bound against the oracle."""
    prob = workloads.make_problem(300, N, 320, seed=71, kind="uniform", bias_mode="row")
    prob.A[:7] = 0.0
    prob.bias[::5] = -0.0
    A, B = dev_operands(prob, "rc")
    bias = prob.bias.cuda()
    fast = ge.gemm_epilogue(A, B, bias, op="bias_relu", bias_mode="row", out_dtype=out_dtype,
                            tile_n=tile_n, cta_group=cg)
    full = bias.view(1, -1).expand(prob.M, -1).contiguous()
    gen = ge.gemm_epilogue(A, B, full, op="bias_relu", bias_mode="full", out_dtype=out_dtype,
                           tile_n=tile_n, cta_group=cg)
    torch.cuda.synchronize()
    bits = torch.int16 if out_dtype == torch.float16 else torch.int32
    assert torch.equal(fast.view(bits), gen.view(bits))
    assert not bool(torch.signbit(fast).any())
    got = fast.float().cpu().numpy().astype(np.float64)
    out, mag = oracle_run(prob, "rc")
    check_bound(got, out, mag, "fast epilogue")


# ------------------------------------------------------------------ multi-GPU sharding, CUDA path (world 1)
@pytest.mark.parametrize("bias_mode", ["row", "col", "full"])
def test_sharded_world1_is_the_batched_call(bias_mode):
    """sharded.py on the CUDA path (no process group: world 1) is the plain batched / single call,
    bitwise, for per-item and shared biases of every mode."""
    from paper_2006_12645_b200 import sharded
    batch, M, N, K = 6, 300, 264, 200
    g = torch.Generator(device="cuda").manual_seed(90)
    U = lambda *s: (torch.rand(*s, generator=g, device="cuda") * 2 - 1).half()
    A, B = U(batch, M, K), U(batch, K, N).transpose(1, 2).contiguous().transpose(1, 2)
    L = {"row": (N,), "col": (M,), "full": (M, N + 8)}[bias_mode]
    for bias in (U(batch, *L), U(*L)):
        got = sharded.sharded_gemm_epilogue_batched(A, B, bias, bias_mode=bias_mode)
        want = ge.gemm_epilogue_batched(A, B, bias, bias_mode=bias_mode)
        torch.cuda.synchronize()
        assert torch.equal(got, want)
    b2 = U(*L)
    got = sharded.sharded_gemm_epilogue_rows(A[0], B[0], b2, bias_mode=bias_mode)
    want = ge.gemm_epilogue(A[0], B[0], b2, bias_mode=bias_mode)
    torch.cuda.synchronize()
    assert torch.equal(got, want)


@pytest.mark.parametrize("layouts", workloads.LAYOUTS)
def test_hadamard_reductions_on_gpu(layouts):
    """S = 1 gives the plain GEMM bitwise; a column-constant S(i,k) = s_k (fp16 values) gives the
    SCALE_K prologue with the same s bitwise (both round fp16(s * a) once: the fp16 x fp16 product is
    exact in fp32); odd K (K tail inside a 16-B chunk) and ld padding of S."""
    prob = workloads.make_problem(300, 264, 203, seed=96, kind="uniform", bias_mode="row")
    A, B = dev_operands(prob, layouts)
    bias = prob.bias.cuda()
    plain = ge.gemm_epilogue(A, B, bias)
    ones = dev_tile(torch.ones(300, 203, dtype=torch.float16), layouts[0], ld=216 if layouts[0] == "r" else 304)
    had1 = ge.gemm_epilogue(A, B, bias, prologue="hadamard", scale=ones)
    s = workloads.uniform_f16((203,), 97, 0.5, 1.5)
    colS = dev_tile(s[None, :].expand(300, 203).contiguous(), layouts[0])
    hadc = ge.gemm_epilogue(A, B, bias, prologue="hadamard", scale=colS)
    sk = ge.gemm_epilogue(A, B, bias, prologue="scale_k", scale=s.float().cuda())
    torch.cuda.synchronize()
    assert torch.equal(had1, plain)
    assert torch.equal(hadc, sk)


def test_hadamard_batched_and_host():
    """Per-item and shared S in the batched call (item b == the single call on item b, bitwise) and
    the host-buffer entry (== the device path, bitwise)."""
    batch, M, N, K = 3, 200, 136, 96
    probs = [workloads.make_problem(M, N, K, seed=800 + b, kind="uniform", bias_mode="row", prologue="hadamard")
             for b in range(batch)]
    A = torch.stack([p.A for p in probs]).cuda()
    B = torch.stack([p.B for p in probs]).cuda()
    S = torch.stack([p.scale for p in probs]).cuda()
    bias = probs[0].bias.cuda()
    for tile in (S, S[1]):
        C = ge.gemm_epilogue_batched(A, B, bias, prologue="hadamard", scale=tile)
        for b in range(batch):
            Cb = ge.gemm_epilogue(A[b], B[b], bias, prologue="hadamard", scale=tile[b] if tile.dim() == 3 else tile)
            torch.cuda.synchronize()
            assert torch.equal(C[b], Cb)
    p0 = probs[0]
    out, mag = oracle_run(p0, "rr")
    got = ge.gemm_epilogue(A[0], B[0], bias, prologue="hadamard", scale=S[0])
    torch.cuda.synchronize()
    check_bound(got.float().cpu().numpy(), out, mag, "hadamard item 0")
    Ch = ge.gemm_epilogue_host(p0.A.pin_memory(), p0.B.pin_memory(), p0.bias.pin_memory(), prologue="hadamard",
                               scale=p0.scale.pin_memory())
    Cd = ge.gemm_epilogue(A[0], B[0], bias, prologue="hadamard", scale=S[0])
    torch.cuda.synchronize()
    assert torch.equal(Ch, Cd.cpu())


# ------------------------------------------------------------------ swap-AB (skinny M)
@pytest.mark.parametrize("layouts", workloads.LAYOUTS)
@pytest.mark.parametrize("bias_mode,op,out_dtype", [("row", "bias_relu", torch.float16), ("col", "bias_relu", torch.float32),
                                                   ("row", "sub_bias_sigmoid", torch.float16), (None, "relu", torch.float16),
                                                   ("row", "literal_bias_relu", torch.float16)])
def test_swap_ab_exact_and_bound(layouts, bias_mode, op, out_dtype):
    """C^T = B^T A^T with a transposed store: forced on a ragged problem (M = 37 rows of C become the
    MMA's N, N = 1000 its 128-row side), on a tile-exact one, on C rows that break the TMA alignment
    (N = 1001: the st.global transposed store) and on a long-K one (split-K clusters under the
    transposed TMA store); ROW and COL bias trade places.  Small integers bitwise, uniform data within
    the bound (sigmoid: bound only)."""
    for M, N, K in ((37, 1000, 200), (64, 256, 128), (37, 1001, 200), (40, 2000, 1024)):
        for kind in ("smallint", "uniform"):
            prob = workloads.make_problem(M, N, K, seed=120, kind=kind, bias_mode=bias_mode or "none")
            assert ge.plan(M, N, K, layouts=layouts, swap_ab=2, bias_mode=bias_mode or "row")["swap_ab"] == 1
            got = run_gpu(prob, layouts, op=op, out_dtype=out_dtype, swap_ab=2)
            act = "sigmoid" if "sigmoid" in op else "relu"
            out, mag = oracle_run(prob, layouts, act=act, bias_sub=op.startswith("sub"),
                                  literal_round=op.startswith("literal"))
            if kind == "smallint" and act == "relu":
                assert np.array_equal(got, exact_expect(out, out_dtype)), (M, N, K, layouts)
            else:
                check_bound(got, out, mag, f"swap {M}x{N}x{K} {layouts}")


def test_swap_ab_batched_padding_and_default():
    """Batched swap-AB (per-item bias), C padding untouched, and the default plan of a skinny
    shape takes the swapped path (BASELINE configs[2] b, scaled down)."""
    assert ge.plan(35, 8457, 2560)["swap_ab"] == 1
    batch, M, N, K = 3, 35, 1030, 136
    probs = [workloads.make_problem(M, N, K, seed=130 + b, kind="smallint", bias_mode="row") for b in range(batch)]
    A = torch.stack([p.A for p in probs]).cuda()
    Bpad = torch.zeros((batch, K, 1032), dtype=torch.float16)        # ldb padded to 16 B (TMA)
    Bpad[:, :, :N] = torch.stack([p.B for p in probs])
    B = Bpad.cuda()[:, :, :N]
    bias = torch.stack([p.bias for p in probs]).cuda()
    Cbuf = torch.full((batch, M, 1040), -5.0, dtype=torch.float16, device="cuda")
    ge.gemm_epilogue_batched(A, B, bias, out=Cbuf[:, :, :N], swap_ab=2)
    torch.cuda.synchronize()
    assert (Cbuf[:, :, N:] == -5.0).all()
    for b, p in enumerate(probs):
        out, _ = oracle_run(p, "rr")
        assert np.array_equal(Cbuf[b, :, :N].float().cpu().numpy().astype(np.float64), exact_expect(out, torch.float16))
    unswapped = ge.gemm_epilogue_batched(A, B, bias, swap_ab=1)
    torch.cuda.synchronize()
    assert torch.equal(unswapped, Cbuf[:, :, :N])          # exact data: both orders agree bitwise


# ------------------------------------------------------------------ half-row CTA pairs (tile_m 128, cta_group 2)
@pytest.mark.parametrize("tile_n", [128, 256])
@pytest.mark.parametrize("layouts", workloads.LAYOUTS)
def test_half_row_pairs_exact_and_bound(tile_n, layouts):
    """cta_group::2 with M = 128 (64 rows per CTA; the accumulator's columns [BN/2, BN) live in TMEM
    lanes 64-127): bitwise on small integers (fp16 and fp32 out) and within the bound + ReLU
    invariant on uniform data, with M/N/K tails (333 x 777 x 321: a partial last row tile of 77 rows,
    i.e. one CTA of the pair with 13 valid rows)."""
    assert ge.plan(333, 777, 321, layouts=layouts, tile_n=tile_n, cta_group=2, tile_m=128)["tile_m"] == 128
    for kind in ("smallint", "uniform"):
        prob = workloads.make_problem(333, 777, 321, seed=140, kind=kind, bias_mode="row")
        for dt in (torch.float16, torch.float32):
            got = run_gpu(prob, layouts, out_dtype=dt, tile_n=tile_n, cta_group=2, tile_m=128)
            pre, mag = oracle_run(prob, layouts, relu=False)
            out = np.where(pre > 0, pre, 0.0)
            if kind == "smallint":
                assert np.array_equal(got, exact_expect(out, dt)), (tile_n, layouts, dt)
            else:
                check_bound(got, out, mag, f"half-row {tile_n} {layouts}")
                check_relu_invariant(got, pre, mag, f"half-row {tile_n} {layouts}")


@pytest.mark.parametrize("variant", ["col_bias", "full_bias", "prologue_scale", "prologue_relu", "hadamard", "batched",
                                     "odd", "k0", "gemm2", "literal"])
def test_half_row_pairs_variants(variant):
    """The half-row pair tile through the other epilogue / prologue / batch paths, bitwise on small
    integers."""
    kw = dict(tile_n=128, cta_group=2, tile_m=128)
    if variant in ("col_bias", "full_bias"):
        bm = "col" if variant == "col_bias" else "full"
        prob = workloads.make_problem(300, 264, 200, seed=141, kind="smallint", bias_mode=bm)
        got = run_gpu(prob, "rc", **kw)
        out, _ = oracle_run(prob, "rc")
        assert np.array_equal(got, exact_expect(out, torch.float16))
    elif variant.startswith("prologue") or variant == "hadamard":
        pro = {"prologue_scale": "scale_k", "prologue_relu": "relu", "hadamard": "hadamard"}[variant]
        for lay in ("rr", "cc"):
            prob = workloads.make_problem(257, 300, 200, seed=142, kind="smallint", bias_mode="row", prologue=pro)
            got = run_gpu(prob, lay, tile_n=256, cta_group=2, tile_m=128)
            out, _ = oracle_run(prob, lay)
            assert np.array_equal(got, exact_expect(out, torch.float16)), (variant, lay)
    elif variant == "batched":
        probs = [workloads.make_problem(200, 136, 96, seed=143 + b, kind="smallint", bias_mode="row") for b in range(3)]
        A = torch.stack([p.A for p in probs]).cuda()
        B = torch.stack([p.B for p in probs]).cuda()
        bias = torch.stack([p.bias for p in probs]).cuda()
        C = ge.gemm_epilogue_batched(A, B, bias, **kw)
        torch.cuda.synchronize()
        for b, p in enumerate(probs):
            out, _ = oracle_run(p, "rr")
            assert np.array_equal(C[b].float().cpu().numpy().astype(np.float64), exact_expect(out, torch.float16))
    elif variant == "odd":
        for (M, N, K) in ((1, 1, 1), (65, 129, 17), (127, 255, 64), (129, 8, 1000)):
            prob = workloads.make_problem(M, N, K, seed=147, kind="smallint", bias_mode="row")
            got = run_gpu(prob, "rr", **kw)
            out, _ = oracle_run(prob, "rr")
            assert np.array_equal(got, exact_expect(out, torch.float16)), (M, N, K)
    elif variant == "k0":
        prob = workloads.make_problem(70, 90, 0, seed=148, bias_mode="col")
        got = run_gpu(prob, "rr", **kw)
        b = prob.bias.float().numpy().astype(np.float64)[:, None] + np.zeros((70, 90))
        assert np.array_equal(got, np.where(b > 0, b, 0.0))
    elif variant == "gemm2":
        p1 = workloads.make_problem(300, 264, 136, seed=149, kind="smallint", bias_mode="row")
        p2 = workloads.make_problem(300, 264, 72, seed=150, kind="smallint", bias_mode=None)
        C = ge.gemm2_epilogue(p1.A.cuda(), p1.B.cuda(), p2.A.cuda(), p2.B.cuda(), p1.bias.cuda(), **kw)
        torch.cuda.synchronize()
        out, _ = oracle.gemm2_epilogue(p1.A, p1.B, p2.A, p2.B, 300, 264, 136, 72, bias=p1.bias, act="relu")
        assert np.array_equal(C.float().cpu().numpy().astype(np.float64), exact_expect(out, torch.float16))
    else:
        prob = _eighths_problem(300, 264, 96, seed=151)
        got = run_gpu(prob, "rr", op="literal_bias_relu", **kw)
        lit, _ = oracle_run(prob, "rr", literal_round=True)
        assert np.array_equal(got, exact_expect(lit, torch.float16))


# ------------------------------------------------------------------ randomized sweep (planner choices)
@pytest.mark.parametrize("chunk", range(8))
def test_random_shapes_bitwise(chunk):
    """A seeded random sweep over shapes (M, N, K in 1..1100 with bias on tile edges, skinny M for
    swap-AB, long K for split-K), the four layouts, bias modes, out dtypes, prologues and ops,
    launched with the DEFAULT plan (whatever tile / split-K / swap-AB / stream-K the planner
    picks): small-integer data is exact in any summation order, so every element must equal
    RNE(oracle) bitwise (fp32 out: the oracle itself)."""
    rng = np.random.default_rng(2026 + chunk)
    for case in range(16):
        kind_shape = rng.integers(0, 4)
        if kind_shape == 0:      # skinny M against a long N (swap-AB territory)
            M, N, K = int(rng.integers(1, 65)), int(rng.integers(1024, 2100)), int(rng.integers(64, 700))
        elif kind_shape == 1:    # few long tiles (split-K territory)
            M, N, K = int(rng.integers(64, 700)), int(rng.integers(64, 300)), int(rng.integers(1500, 4000))
        else:
            M, N, K = (int(x) for x in rng.integers(1, 1100, size=3))
        layouts = str(rng.choice(workloads.LAYOUTS))
        bias_mode = str(rng.choice(["row", "col", "full", "none"]))
        out_dtype = torch.float32 if rng.random() < 0.3 else torch.float16
        prologue = str(rng.choice(["none", "none", "scale_k", "relu"])) if bias_mode != "none" else "none"
        prob = workloads.make_problem(M, N, K, seed=3000 + 100 * chunk + case, kind="smallint",
                                      bias_mode=bias_mode, prologue=None if prologue == "none" else prologue)
        what = (M, N, K, layouts, bias_mode, str(out_dtype), prologue)
        got = run_gpu(prob, layouts, out_dtype=out_dtype, op=None if bias_mode != "none" else "relu")
        out, _ = oracle_run(prob, layouts)
        assert np.array_equal(got, exact_expect(out, out_dtype)), what
