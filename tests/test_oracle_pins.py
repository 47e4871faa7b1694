"""Pins for the CPU oracle (oracle/ge_oracle.c) against things other than itself:
numpy's fp16 codec, hand-computed golden cases (tests/golden/hand_cases.json),
exact rational brute force, numpy fp64 matmul, and closed forms.  Each test
names the passage of PAPER.md (or the DESIGN.md reading) it pins.  CPU only."""
from __future__ import annotations

import itertools
import json
import os
from fractions import Fraction

import numpy as np
import pytest
import torch

import oracle
import workloads
from tests.helpers import oracle_run

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "hand_cases.json")


# ---------------------------------------------------------------- fp16 codec
def test_decode_all_patterns_vs_numpy():
    """Oracle's own fp16 decoder == numpy float16 widening, all 65536 patterns (IEEE 754 binary16)."""
    bits = np.arange(65536, dtype=np.uint16)
    ours = oracle.f16_decode(bits)
    ref = bits.view(np.float16).astype(np.float64)
    nan = np.isnan(ref)
    assert np.array_equal(np.isnan(ours), nan)
    assert np.array_equal(ours[~nan], ref[~nan])
    assert np.array_equal(np.signbit(ours[~nan]), np.signbit(ref[~nan]))


def test_encode_rne_vs_numpy():
    """Oracle's RNE fp64->fp16 encoder == numpy's correctly rounded double->half, incl. ties,
    subnormals and overflow (DESIGN.md R-C6)."""
    rng = np.random.default_rng(0)
    xs = [rng.uniform(-1, 1, 20000) * 10.0 ** rng.integers(-9, 5, 20000)]
    # exact ties between adjacent fp16 values, across binades and the subnormal range
    h = rng.integers(0, 0x7bff, 20000).astype(np.uint16)
    lo = h.view(np.float16).astype(np.float64)
    hi = (h + 1).view(np.float16).astype(np.float64)
    xs.append((lo + hi) / 2)
    xs.append(-(lo + hi) / 2)
    xs.append(np.array([0.0, -0.0, 1.0, 2049.0, 2050.0, 2051.0, 65504.0, 65519.99, 65520.0, 1e6, -1e6,
                        2.0 ** -24, 2.0 ** -25, 3 * 2.0 ** -25, 2.0 ** -26, 2.0 ** -14, 2.0 ** -14 - 2.0 ** -25,
                        np.inf, -np.inf]))
    x = np.concatenate(xs)
    ours = oracle.f16_encode(x)
    with np.errstate(over="ignore"):
        ref = x.astype(np.float16).view(np.uint16)
    assert np.array_equal(ours, ref)


def test_codec_spec_points():
    """SPEC.md:568-570 pins: 1.0 <-> 0x3C00, 2049 -> 2048 (tie to even), 65520 -> +inf, 2^-24 round trip."""
    enc = oracle.f16_encode(np.array([1.0, 2049.0, 65520.0, 2.0 ** -24]))
    assert list(enc) == [0x3C00, 0x6800, 0x7C00, 0x0001]
    assert list(oracle.f16_decode(np.array([0x3C00, 0x0001], dtype=np.uint16))) == [1.0, 2.0 ** -24]


# ---------------------------------------------------------------- golden
def _golden_cases():
    with open(GOLDEN) as f:
        return json.load(f)["cases"]


@pytest.mark.parametrize("case", _golden_cases(), ids=lambda c: c["name"])
@pytest.mark.parametrize("layouts", workloads.LAYOUTS)
def test_hand_computed_cases(case, layouts):
    M, N, K = case["M"], case["N"], case["K"]
    A = torch.tensor(case["A"], dtype=torch.float16).reshape(M, K)
    B = torch.tensor(case["B"], dtype=torch.float16).reshape(K, N)
    bias = None if case["bias"] is None else torch.tensor(case["bias"], dtype=torch.float16)
    scale = None if case.get("scale") is None else torch.tensor(case["scale"], dtype=torch.float32)
    if case["prologue"] == "hadamard":
        scale = torch.tensor(case["S"], dtype=torch.float16).reshape(M, K)
    prob = workloads.Problem(M, N, K, A, B, bias, scale,
                             {"bias_mode": case["bias_mode"], "prologue": case["prologue"]})
    out, mag = oracle_run(prob, layouts, relu=case["relu"], literal_round=case.get("literal_round", False))
    assert np.array_equal(out, np.array(case["out"], dtype=np.float64).reshape(M, N))
    assert np.array_equal(mag, np.array(case["mag"], dtype=np.float64).reshape(M, N))
    assert not np.signbit(out[out == 0]).any() or not case["relu"]


def test_literal_golden_cases_reject_wrong_rounding_points():
    """Negative controls for the literal-rounding pins (DESIGN.md R-C3): on the
    hand-computed literal cases, an evaluation that rounds once (f16(acc + beta)), or that skips
    either of the two roundings, must disagree with the golden value in at least one case each."""
    lit = [c for c in _golden_cases() if c.get("literal_round")]
    assert len(lit) >= 4
    f16 = lambda x: oracle.f16_decode(oracle.f16_encode(np.asarray(x, dtype=np.float64)))
    miss = {"single (no first rounding)": 0, "no second rounding": 0, "no rounding": 0}
    for c in lit:
        M, N, K = c["M"], c["N"], c["K"]
        A = np.array(c["A"], dtype=np.float64).reshape(M, K)
        B = np.array(c["B"], dtype=np.float64).reshape(K, N)
        acc = A @ B                                  # exact: small integers and powers of two
        b = np.array(c["bias"], dtype=np.float64)
        beta = b[None, :] if c["bias_mode"] == "row" else b[:, None]
        relu = (lambda v: np.where(v > 0, v, 0.0)) if c["relu"] else (lambda v: v)
        want = np.array(c["out"], dtype=np.float64).reshape(M, N)
        miss["single (no first rounding)"] += not np.array_equal(relu(f16(acc + beta)), want)
        miss["no second rounding"] += not np.array_equal(relu(f16(acc) + beta), want)
        miss["no rounding"] += not np.array_equal(relu(acc + beta), want)
        # and the golden value is what the two-rounding definition gives (consistency of the file)
        assert np.array_equal(relu(f16(f16(acc) + beta)), want), c["name"]
    assert all(v >= 1 for v in miss.values()), miss


# ---------------------------------------------------------------- brute force, exact rationals
def _exact(prob, relu, bias_mode):
    A = [[Fraction(float(v)) for v in row] for row in prob.A.float().tolist()]
    B = [[Fraction(float(v)) for v in row] for row in prob.B.float().tolist()]
    if prob.meta.get("prologue") == "scale_k":
        s = [Fraction(float(v)) for v in prob.scale.tolist()]
        A = [[s[k] * A[i][k] for k in range(prob.K)] for i in range(prob.M)]
    elif prob.meta.get("prologue") == "hadamard":
        S = [[Fraction(float(v)) for v in row] for row in prob.scale.float().tolist()]
        A = [[S[i][k] * A[i][k] for k in range(prob.K)] for i in range(prob.M)]
    elif prob.meta.get("prologue") == "relu":
        A = [[max(v, Fraction(0)) for v in row] for row in A]
    outs, mags = [], []
    for i in range(prob.M):
        ro, rm = [], []
        for j in range(prob.N):
            acc = sum((A[i][k] * B[k][j] for k in range(prob.K)), Fraction(0))
            mg = sum((abs(A[i][k] * B[k][j]) for k in range(prob.K)), Fraction(0))
            if bias_mode == "row":
                acc += Fraction(float(prob.bias[j]))
            elif bias_mode == "col":
                acc += Fraction(float(prob.bias[i]))
            elif bias_mode == "full":
                acc += Fraction(float(prob.bias[i, j]))
            if relu and acc <= 0:
                acc = Fraction(0)
            ro.append(acc)
            rm.append(mg)
        outs.append(ro)
        mags.append(rm)
    return outs, mags


def test_brute_force_exact_rationals():
    """Every (M,N,K) in {1,2,3,5,8}^3 against an exact rational evaluation of Listing 1 / Listing 5
    (PAPER.md:355-364, 1201-1206): |oracle - exact| <= 1e-12 * mag (fp64 summation)."""
    dims = (1, 2, 3, 5, 8)
    modes = ("row", "col", "full", None)
    pros = (None, "relu", "scale_k", "hadamard")
    for n, (M, N, K) in enumerate(itertools.product(dims, dims, dims)):
        bm, pro, lay = modes[n % 4], pros[(n // 4) % 4], workloads.LAYOUTS[n % 4]
        relu = n % 2 == 0
        prob = workloads.make_problem(M, N, K, seed=1000 + n, bias_mode=bm, prologue=pro)
        out, mag = oracle_run(prob, lay, relu=relu)
        eo, em = _exact(prob, relu, bm)
        for i in range(M):
            for j in range(N):
                assert abs(Fraction(out[i, j]) - eo[i][j]) <= Fraction(1e-12) * em[i][j] + Fraction(0), \
                    (M, N, K, i, j, out[i, j], float(eo[i][j]))
                assert abs(Fraction(mag[i, j]) - em[i][j]) <= Fraction(1e-12) * em[i][j]


# ---------------------------------------------------------------- numpy cross-check
def _numpy_ref(prob, relu):
    A = prob.A.numpy().astype(np.float64)
    B = prob.B.numpy().astype(np.float64)
    pre = A @ B
    mag = np.abs(A) @ np.abs(B)
    bm = prob.meta["bias_mode"]
    if bm == "row":
        pre = pre + prob.bias.numpy().astype(np.float64)[None, :]
    elif bm == "col":
        pre = pre + prob.bias.numpy().astype(np.float64)[:, None]
    elif bm == "full":
        pre = pre + prob.bias.numpy().astype(np.float64)[:, :prob.N]
    return (np.where(pre > 0, pre, 0.0) if relu else pre), mag


@pytest.mark.parametrize("layouts", workloads.LAYOUTS)
@pytest.mark.parametrize("bias_mode", ["row", "col", "full"])
def test_numpy_fp64_crosscheck(layouts, bias_mode):
    """Oracle vs numpy float64 matmul on the same widened inputs (ragged 300x520x200)."""
    prob = workloads.make_problem(300, 520, 200, seed=5, bias_mode=bias_mode)
    out, mag = oracle_run(prob, layouts)
    ref, rmag = _numpy_ref(prob, True)
    assert np.all(np.abs(out - ref) <= 1e-12 * rmag + 1e-300)
    assert np.allclose(mag, rmag, rtol=1e-12, atol=0)


def test_negative_controls_fail():
    """A deliberately broken evaluation (transposed B, dropped bias) must fail the cross-check,
    proving the check can see those mistakes (SPEC.md:210, 616 negative-control idea)."""
    prob = workloads.make_problem(64, 64, 64, seed=9, bias_mode="row")
    ref, rmag = _numpy_ref(prob, True)
    Bs, _ = workloads.store(prob.B, "r")
    As, _ = workloads.store(prob.A, "r")
    wrong, _ = oracle.gemm_epilogue(As, Bs, 64, 64, 64, layoutA="row", layoutB="col", bias=prob.bias)
    assert not np.all(np.abs(wrong - ref) <= 1e-12 * rmag)
    nobias, _ = oracle.gemm_epilogue(As, Bs, 64, 64, 64, layoutA="row", layoutB="row", bias=None)
    assert not np.all(np.abs(nobias - ref) <= 1e-12 * rmag)


# ---------------------------------------------------------------- closed forms
@pytest.mark.parametrize("layouts", workloads.LAYOUTS)
def test_identity(layouts):
    """A = I (a(i,k) = [i=k]) => out = relu(b(i,j)[i<K] + bias[j]), exact."""
    M, N, K = 70, 50, 40
    prob = workloads.make_problem(M, N, K, seed=11, bias_mode="row")
    prob.A = torch.eye(M, K, dtype=torch.float16)
    out, _ = oracle_run(prob, layouts)
    b = np.zeros((M, N))
    b[:K] = prob.B.numpy().astype(np.float64)
    pre = b + prob.bias.numpy().astype(np.float64)[None, :]
    assert np.array_equal(out, np.where(pre > 0, pre, 0.0))


@pytest.mark.parametrize("layouts", workloads.LAYOUTS)
def test_all_ones(layouts):
    """a = b = 1 => pre = K + bias (integer bias), exact."""
    M, N, K = 33, 65, 129
    prob = workloads.make_problem(M, N, K, seed=12, kind="smallint", bias_mode="col")
    prob.A = torch.ones(M, K, dtype=torch.float16)
    prob.B = torch.ones(K, N, dtype=torch.float16)
    out, mag = oracle_run(prob, layouts, relu=False)
    assert np.array_equal(out, K + prob.bias.numpy().astype(np.float64)[:, None] + np.zeros((M, N)))
    assert np.array_equal(mag, np.full((M, N), float(K)))


@pytest.mark.parametrize("layouts", workloads.LAYOUTS)
def test_diagonal(layouts):
    """A = diag(d) => pre = d_i * b(i,j) + bias[i,j] (FULL bias), exact in fp64."""
    M = N = K = 48
    prob = workloads.make_problem(M, N, K, seed=13, bias_mode="full")
    d = workloads.uniform_f16((M,), 77)
    prob.A = torch.diag(d)
    out, _ = oracle_run(prob, layouts)
    pre = d.numpy().astype(np.float64)[:, None] * prob.B.numpy().astype(np.float64) \
        + prob.bias.numpy().astype(np.float64)
    assert np.array_equal(out, np.where(pre > 0, pre, 0.0))


@pytest.mark.parametrize("layouts", workloads.LAYOUTS)
def test_rank1_powers_of_two(layouts):
    """a(i,k) = 2^p_i, b(k,j) = 2^q_j => pre = K * 2^(p_i+q_j), exact."""
    M, N, K = 20, 24, 64
    g = workloads.gen(14)
    p = torch.randint(-6, 4, (M,), generator=g)
    q = torch.randint(-6, 4, (N,), generator=g)
    A = torch.pow(2.0, p.double())[:, None].expand(M, K).to(torch.float16)
    B = torch.pow(2.0, q.double())[None, :].expand(K, N).to(torch.float16)
    prob = workloads.Problem(M, N, K, A, B, None, None, {"bias_mode": None, "prologue": None})
    out, _ = oracle_run(prob, layouts, relu=False)
    assert np.array_equal(out, K * np.exp2((p[:, None] + q[None, :]).double().numpy()))


def test_zeros_and_k0():
    """A = 0 or K = 0 => out = op(beta) (DESIGN.md R-C9), for each bias mode with distinct values."""
    for bm in ("row", "col", "full"):
        for K in (0, 17):
            prob = workloads.make_problem(9, 11, K, seed=15, bias_mode=bm)
            prob.A = torch.zeros(9, K, dtype=torch.float16)
            out, mag = oracle_run(prob, "rc")
            bias = prob.bias.numpy().astype(np.float64)
            if bm == "row":
                beta = bias[None, :] + np.zeros((9, 11))
            elif bm == "col":
                beta = bias[:, None] + np.zeros((9, 11))
            else:
                beta = bias[:, :11]
            assert np.array_equal(out, np.where(beta > 0, beta, 0.0))
            assert not mag.any()


# ---------------------------------------------------------------- invariants
def test_layout_invariance_bitwise():
    """The same logical A, B in rr/rc/cr/cc give bitwise-identical oracle outputs (PAPER.md:609-610:
    the four layout specialisations compute the same product)."""
    prob = workloads.make_problem(37, 45, 53, seed=16, bias_mode="row")
    outs = [oracle_run(prob, lay)[0] for lay in workloads.LAYOUTS]
    for o in outs[1:]:
        assert np.array_equal(o, outs[0])


def test_padded_leading_dims():
    """Explicit lda/ldb larger than packed (PAPER.md:844 carries ldM_0/ldM_1) give the same result."""
    prob = workloads.make_problem(30, 40, 50, seed=17, bias_mode="row")
    base = oracle_run(prob, "cr")[0]
    padded = oracle_run(prob, "cr", lda=64, ldb=48)[0]
    assert np.array_equal(base, padded)


def test_relu_invariant():
    """relu at the root of relu_add: out >= 0, out == 0 exactly where pre <= 0,
    out == pre where pre > 0, and zeros are +0 (DESIGN.md R-C5)."""
    prob = workloads.make_problem(64, 96, 80, seed=18, bias_mode="row")
    pre, _ = oracle_run(prob, "rr", relu=False)
    out, _ = oracle_run(prob, "rr", relu=True)
    assert (out >= 0).all() and not np.signbit(out).any()
    assert np.array_equal(out[pre <= 0], np.zeros(int((pre <= 0).sum())))
    assert np.array_equal(out[pre > 0], pre[pre > 0])
    assert 0.2 < (pre <= 0).mean() < 0.8     # the recipe exercises both branches


def test_prologue_identities():
    """Prologue pins (DESIGN.md R-C12): s == 1 is NONE bitwise; s == 4 scales the
    bias-free pre-activation by exactly 4; RELU prologue == NONE on a pre-clamped copy of A."""
    prob = workloads.make_problem(40, 56, 72, seed=19, bias_mode=None)
    none = oracle_run(prob, "rr", relu=False)[0]
    p1 = workloads.Problem(prob.M, prob.N, prob.K, prob.A, prob.B, None, torch.ones(prob.K),
                           {"bias_mode": None, "prologue": "scale_k"})
    assert np.array_equal(oracle_run(p1, "rr", relu=False)[0], none)
    p4 = workloads.Problem(prob.M, prob.N, prob.K, prob.A, prob.B, None, torch.full((prob.K,), 4.0),
                           {"bias_mode": None, "prologue": "scale_k"})
    assert np.array_equal(oracle_run(p4, "cc", relu=False)[0], 4.0 * none)
    pr = workloads.Problem(prob.M, prob.N, prob.K, prob.A, prob.B, None, None,
                           {"bias_mode": None, "prologue": "relu"})
    clamped = workloads.Problem(prob.M, prob.N, prob.K, torch.clamp(prob.A, min=0), prob.B, None, None,
                                {"bias_mode": None, "prologue": None})
    assert np.array_equal(oracle_run(pr, "cr", relu=False)[0], oracle_run(clamped, "cr", relu=False)[0])


def test_sampled_rows_cols_match_full():
    """The row/column-sampled evaluation returns exactly the entries of the full evaluation."""
    prob = workloads.make_problem(50, 70, 30, seed=20, bias_mode="full")
    full, fmag = oracle_run(prob, "rc")
    rows, cols = [0, 7, 49, 7], [69, 0, 33]
    sub, smag = oracle_run(prob, "rc", rows=rows, cols=cols)
    assert np.array_equal(sub, full[np.ix_(rows, cols)])
    assert np.array_equal(smag, fmag[np.ix_(rows, cols)])


def test_smallint_exactness_and_literal_reading():
    """Small-integer data is exact in fp64 and fp32 in any order (|partial sums| < 2^23), and the
    paper-literal rounding (DESIGN.md R-C3: relu(f16(f16(acc)+bias))) stays within the bound."""
    prob = workloads.make_problem(64, 64, 512, seed=21, kind="smallint", bias_mode="row")
    out, mag = oracle_run(prob, "rr")
    ref, _ = _numpy_ref(prob, True)
    assert np.array_equal(out, ref)
    assert np.array_equal(out, np.round(out))
    uprob = workloads.make_problem(64, 64, 512, seed=22, bias_mode="row")
    o, m = oracle_run(uprob, "rr")
    lit, _ = oracle_run(uprob, "rr", literal_round=True)
    assert np.all(np.abs(lit - o) <= oracle.bound(o, m))
    assert not np.array_equal(lit, o)      # the two readings really differ


def test_bad_arguments_rejected():
    with pytest.raises(ValueError):
        oracle.gemm_epilogue(np.zeros(4, np.uint16), np.zeros(4, np.uint16), 2, 2, 2, bias=None,
                             rows=[5], cols=[0])


# ---------------------------------------------------------------- the paper's pointwise op set
# add, subtract, ReLU, Sigmoid, Tanh.  Pinned by special values and
# identities the mathematics fixes (not by retyping the formulas).
def _prob_nobias(M=48, N=40, K=32, seed=60):
    return workloads.make_problem(M, N, K, seed=seed, bias_mode=None)


def _run(prob, A=None, act=None, bias=None, bias_sub=False, layouts="rc"):
    p = workloads.Problem(prob.M, prob.N, prob.K, prob.A if A is None else A, prob.B, bias, None,
                          {"bias_mode": "row" if bias is not None else None, "prologue": None})
    As, lda = workloads.store(p.A, layouts[0])
    Bs, ldb = workloads.store(p.B, layouts[1])
    return oracle.gemm_epilogue(As, Bs, p.M, p.N, p.K, layoutA="row" if layouts[0] == "r" else "col",
                                layoutB="row" if layouts[1] == "r" else "col", lda=lda, ldb=ldb,
                                bias=bias, bias_mode="row", act=act, bias_sub=bias_sub)[0]


def test_sigmoid_tanh_at_zero():
    """sigma(0) = 1/2 and tanh(0) = 0 exactly (A = 0: pre-activation is exactly 0)."""
    prob = _prob_nobias()
    Z = torch.zeros_like(prob.A)
    assert np.all(_run(prob, A=Z, act="sigmoid") == 0.5)
    assert np.all(_run(prob, A=Z, act="tanh") == 0.0)


def test_sigmoid_tanh_symmetries():
    """sigma(-x) = 1 - sigma(x), tanh(-x) = -tanh(x): negating A negates pre exactly."""
    prob = _prob_nobias()
    for act, check in (("sigmoid", lambda a, b: np.abs(a + b - 1.0).max() < 1e-15),
                       ("tanh", lambda a, b: np.abs(a + b).max() < 1e-15)):
        assert check(_run(prob, act=act), _run(prob, A=-prob.A, act=act))


def test_tanh_sigmoid_identity():
    """tanh(x) = 2*sigma(2x) - 1 ties the two independent implementations; 2A is exact in fp16."""
    prob = _prob_nobias()
    t = _run(prob, act="tanh")
    s2 = _run(prob, A=prob.A * 2, act="sigmoid")
    assert np.abs(t - (2 * s2 - 1)).max() < 1e-14
    assert 0.0 < s2.min() and s2.max() < 1.0


def test_sigmoid_monotone_in_pre():
    """The activation is applied to the same pre-activation: its order is preserved."""
    prob = _prob_nobias(seed=61)
    pre = _run(prob, act=None)
    for act in ("sigmoid", "tanh"):
        y = _run(prob, act=act)
        o = np.argsort(pre.ravel(), kind="stable")
        assert np.all(np.diff(y.ravel()[o]) >= 0)


@pytest.mark.parametrize("act", [None, "relu", "sigmoid", "tanh"])
def test_subtract_bias_is_add_of_negated_bias(act):
    """A - bias == A + (-bias) bitwise (fp16 negation is exact) for every activation."""
    prob = workloads.make_problem(37, 45, 53, seed=62, bias_mode="row")
    a = _run(prob, act=act, bias=prob.bias, bias_sub=True)
    b = _run(prob, act=act, bias=-prob.bias, bias_sub=False)
    assert np.array_equal(a, b)
    assert not np.array_equal(a, _run(prob, act=act, bias=prob.bias)) or act == "relu"


# ---------------------------------------------------------------- sum of matmuls (Listing 4)
def test_gemm2_golden_and_block_identity():
    """Hand case: 1*2 + 3*4 - 4 = 10 (PAPER.md:1157-1166, S3 add then relu_add); and the block
    identity A.B + P.Q = [A P].[B; Q] against the single-GEMM oracle on concatenated operands."""
    one = lambda v: torch.tensor([[v]], dtype=torch.float16)
    out, mag = oracle.gemm2_epilogue(one(1), one(2), one(3), one(4), 1, 1, 1, 1, bias=torch.tensor([-4.0]).half(),
                                     bias_mode="row", act="relu")
    assert out[0, 0] == 10.0 and mag[0, 0] == 14.0
    M, N, K1, K2 = 40, 56, 48, 24
    p1 = workloads.make_problem(M, N, K1, seed=70, bias_mode="col")
    p2 = workloads.make_problem(M, N, K2, seed=71, bias_mode=None)
    z, zm = oracle.gemm2_epilogue(p1.A, p1.B, p2.A, p2.B, M, N, K1, K2, bias=p1.bias, bias_mode="col", act="tanh")
    cat = workloads.Problem(M, N, K1 + K2, torch.cat([p1.A, p2.A], 1), torch.cat([p1.B, p2.B], 0), p1.bias, None,
                            {"bias_mode": "col", "prologue": None})
    ref, rm = oracle_run(cat, "rr", act="tanh")
    assert np.all(np.abs(z - ref) <= 1e-12 * (rm + 1))
    assert np.allclose(zm, rm, rtol=1e-12)


def test_gemm2_reductions():
    """P = 0 reduces to the single GEMM (bitwise); swapping the two products commutes (bitwise)."""
    M, N, K1, K2 = 33, 47, 40, 16
    p1 = workloads.make_problem(M, N, K1, seed=72, bias_mode="row")
    p2 = workloads.make_problem(M, N, K2, seed=73, bias_mode=None)
    z0, _ = oracle.gemm2_epilogue(p1.A, p1.B, torch.zeros(M, K2, dtype=torch.float16), p2.B, M, N, K1, K2,
                                  bias=p1.bias, act="relu")
    single, _ = oracle_run(p1, "rr")
    assert np.array_equal(z0, single)
    pb = workloads.make_problem(M, N, K1, seed=74, bias_mode=None)
    a, _ = oracle.gemm2_epilogue(p1.A, p1.B, pb.A, pb.B, M, N, K1, K1, bias=p1.bias, act=None)
    b, _ = oracle.gemm2_epilogue(pb.A, pb.B, p1.A, p1.B, M, N, K1, K1, bias=p1.bias, act=None)
    assert np.array_equal(a, b)


# ---------------------------------------------------------------- Hadamard prologue (R-C18)
def _had(prob, S):
    return workloads.Problem(prob.M, prob.N, prob.K, prob.A, prob.B, prob.bias, S,
                             {"bias_mode": prob.meta["bias_mode"], "prologue": "hadamard"})


@pytest.mark.parametrize("layouts", workloads.LAYOUTS)
def test_hadamard_special_cases(layouts):
    """Full-tile Hadamard prologue a'(i,k) = s(i,k) a(i,k) (DESIGN.md R-C18), pinned
    by reductions the mathematics fixes: S = 1 is the plain GEMM bitwise; S = 2^p scales the bias-free
    pre-activation by exactly 2^p; a per-row S(i,k) = 2^p_i scales row i by 2^p_i (a transposed S
    fails this); a per-column S(i,k) = s_k is the (already pinned) SCALE_K prologue bitwise."""
    M, N, K = 37, 45, 53
    prob = workloads.make_problem(M, N, K, seed=95, bias_mode=None)
    none = oracle_run(prob, layouts, relu=False)[0]
    assert np.array_equal(oracle_run(_had(prob, torch.ones(M, K, dtype=torch.float16)), layouts, relu=False)[0], none)
    assert np.array_equal(oracle_run(_had(prob, torch.full((M, K), 0.25, dtype=torch.float16)), layouts,
                                     relu=False)[0], 0.25 * none)
    p = torch.randint(-3, 4, (M,), generator=workloads.gen(96))
    rowS = torch.pow(2.0, p.double())[:, None].expand(M, K).to(torch.float16)
    got = oracle_run(_had(prob, rowS), layouts, relu=False)[0]
    assert np.array_equal(got, np.exp2(p.double().numpy())[:, None] * none)
    # control: the same exponents applied along k instead of i do not give the row-scaled result
    q = torch.randint(-3, 4, (K,), generator=workloads.gen(99))
    kS = torch.pow(2.0, q.double())[None, :].expand(M, K).to(torch.float16)
    assert not np.array_equal(oracle_run(_had(prob, kS), layouts, relu=False)[0], got)
    s = workloads.uniform_f16((K,), 97, 0.5, 1.5)
    colS = s[None, :].expand(M, K).contiguous()
    sk = workloads.Problem(M, N, K, prob.A, prob.B, None, s.float(), {"bias_mode": None, "prologue": "scale_k"})
    assert np.array_equal(oracle_run(_had(prob, colS), layouts, relu=False)[0], oracle_run(sk, layouts, relu=False)[0])


def test_hadamard_numpy_crosscheck():
    """(A * S) @ B + bias, relu, in numpy fp64 on a ragged shape, every layout of A (S follows A)."""
    prob = workloads.make_problem(70, 90, 110, seed=98, bias_mode="row", prologue="hadamard")
    A = prob.A.numpy().astype(np.float64) * prob.scale.numpy().astype(np.float64)
    B = prob.B.numpy().astype(np.float64)
    pre = A @ B + prob.bias.numpy().astype(np.float64)[None, :]
    ref, rmag = np.where(pre > 0, pre, 0.0), np.abs(A) @ np.abs(B)
    for lay in workloads.LAYOUTS:
        out, mag = oracle_run(prob, lay)
        assert np.all(np.abs(out - ref) <= 1e-12 * rmag + 1e-300), lay
        assert np.allclose(mag, rmag, rtol=1e-12, atol=0)
