"""Shared test helpers: run the oracle on a workloads.Problem in a given layout,
and the per-element acceptance check of BASELINE.json's north_star."""
from __future__ import annotations

import numpy as np
import torch

import oracle
import workloads


def stored(prob: workloads.Problem, layouts: str, lda=None, ldb=None):
    """Storage tensors (CPU fp16) and leading dims of A and B for layout pair e.g. 'rc'."""
    As, lda = workloads.store(prob.A, layouts[0], lda)
    Bs, ldb = workloads.store(prob.B, layouts[1], ldb)
    return As, lda, Bs, ldb


def oracle_run(prob: workloads.Problem, layouts: str = "rr", *, relu=True, bias_mode=None, rows=None,
               cols=None, literal_round=False, lda=None, ldb=None, nthreads=None, act="default", bias_sub=False):
    bias_mode = prob.meta.get("bias_mode") if bias_mode is None else bias_mode
    As, lda, Bs, ldb = stored(prob, layouts, lda, ldb)
    ldbias = prob.bias.shape[1] if (prob.bias is not None and prob.bias.dim() == 2) else 0
    pro = prob.meta.get("prologue")
    scale, lds = prob.scale, None
    if pro == "hadamard":          # the tile S is stored in A's layout
        scale, lds = workloads.store(prob.scale, layouts[0])
    return oracle.gemm_epilogue(
        As, Bs, prob.M, prob.N, prob.K,
        layoutA="row" if layouts[0] == "r" else "col", layoutB="row" if layouts[1] == "r" else "col",
        lda=lda, ldb=ldb, bias=prob.bias, bias_mode=bias_mode if prob.bias is not None else None,
        ldbias=ldbias, relu=relu, act=act, bias_sub=bias_sub, prologue=pro, scale=scale, lds=lds,
        literal_round=literal_round, rows=rows, cols=cols, nthreads=nthreads)


def check_bound(got: np.ndarray, out: np.ndarray, mag: np.ndarray, what: str = ""):
    """|got - out| <= 4e-3*mag + 1e-3*|out| element-wise (BASELINE.json north_star).
    A 2^-25 absolute slack covers fp16 subnormal outputs with tiny mag (DESIGN.md R-TOL)."""
    got = np.asarray(got, dtype=np.float64)
    tol = oracle.bound(out, mag) + 2.0 ** -25
    err = np.abs(got - out)
    bad = ~(err <= tol)
    if bad.any():
        idx = np.argwhere(bad)[:5]
        msg = "; ".join(f"{tuple(i)} got={got[tuple(i)]!r} want={out[tuple(i)]!r} tol={tol[tuple(i)]:.3g}"
                        for i in idx)
        raise AssertionError(f"{what}: {int(bad.sum())} / {bad.size} elements outside the bound: {msg}")
    return float(np.max(err / np.maximum(tol, 1e-300))) if err.size else 0.0


def f16_bits(t: torch.Tensor) -> np.ndarray:
    return t.detach().cpu().contiguous().view(torch.int16).numpy().view(np.uint16)


def check_relu_invariant(got: np.ndarray, pre: np.ndarray, mag: np.ndarray, what: str = ""):
    """BASELINE.json north_star ReLU invariant on the GPU output, given the oracle's unrounded
    pre-activation: every value is >= 0, finite and not -0 (DESIGN.md R-C5); it is exactly +0
    wherever pre <= -tol, and > 0 wherever pre >= tol and RNE_fp16(pre) > 0 (tol = the per-element
    bound; the band |pre| < tol is where rounding may legitimately decide the sign).
    Returns (#forced zeros, #forced positives) so callers can assert both branches were exercised."""
    got = np.asarray(got, dtype=np.float64)
    tol = oracle.bound(pre, mag) + 2.0 ** -25
    assert np.isfinite(got).all(), f"{what}: non-finite output"
    assert (got >= 0).all(), f"{what}: negative output after ReLU"
    assert not np.signbit(got).any(), f"{what}: -0 in the output (ReLU must give +0)"
    neg = pre <= -tol
    assert (got[neg] == 0).all(), f"{what}: {int((got[neg] != 0).sum())} nonzero outputs where pre <= -tol"
    pos = (pre >= tol) & (oracle.f16_decode(oracle.f16_encode(pre)) > 0)
    assert (got[pos] > 0).all(), f"{what}: {int((got[pos] <= 0).sum())} zero outputs where pre >= tol"
    return int(neg.sum()), int(pos.sum())
