"""Seeded synthetic inputs shared by the tests, smoke() and bench.py.

This module holds NO arithmetic of the method: it only draws seeded random
numbers and lays logical matrices out in memory (row- or column-major storage
with a leading dimension).  Both the oracle and the CUDA path consume what it
produces; neither side imports the other.

Input recipe: the paper gives sizes only (PAPER.md:1249-1252,
"problem sizes being multiples of 128 up to 4096"), so values are ours:
  * "uniform": A, B, bias ~ U(-1, 1) drawn as fp32 by a CPU torch.Generator(seed),
    then rounded to fp16 (RNE) -> identical bits on every machine.
  * "smallint": a, b ~ U{-3..3}, bias ~ U{-8..8} (exact-arithmetic pin).
  * prologue scale s ~ U(0.5, 1.5) fp32 (uniform) or s in {0.5, 1, 2} (smallint).
  * Hadamard prologue tile S (M x K fp16): U(0.5, 1.5) rounded to fp16 (uniform) or
    S in {-1, 0.5, 1, 2} (smallint: every a*s is exact in fp16 and the sums stay exact in fp32).
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Optional

import torch

LAYOUTS = ("rr", "rc", "cr", "cc")  # (layout of A, layout of B): r = row-major, c = col-major


def gen(seed: int) -> torch.Generator:
    g = torch.Generator(device="cpu")
    g.manual_seed(int(seed))
    return g


def uniform_f16(shape, seed: int, lo: float = -1.0, hi: float = 1.0) -> torch.Tensor:
    g = gen(seed)
    return (torch.rand(shape, generator=g, dtype=torch.float32) * (hi - lo) + lo).to(torch.float16)


def smallint_f16(shape, seed: int, lo: int = -3, hi: int = 3) -> torch.Tensor:
    g = gen(seed)
    return torch.randint(lo, hi + 1, shape, generator=g, dtype=torch.int32).to(torch.float16)


def scale_vector(K: int, seed: int, kind: str = "uniform") -> torch.Tensor:
    g = gen(seed)
    if kind == "smallint":
        choices = torch.tensor([0.5, 1.0, 2.0], dtype=torch.float32)
        return choices[torch.randint(0, 3, (K,), generator=g)]
    return torch.rand((K,), generator=g, dtype=torch.float32) + 0.5


def hadamard_tile(M: int, K: int, seed: int, kind: str = "uniform") -> torch.Tensor:
    """Logical M x K fp16 tile S of the Hadamard prologue (a'(i,k) = S[i,k] * A[i,k])."""
    g = gen(seed)
    if kind == "smallint":
        choices = torch.tensor([-1.0, 0.5, 1.0, 2.0], dtype=torch.float32)
        return choices[torch.randint(0, 4, (M, K), generator=g)].to(torch.float16)
    return (torch.rand((M, K), generator=g, dtype=torch.float32) + 0.5).to(torch.float16)


def store(logical: torch.Tensor, layout: str, ld: Optional[int] = None) -> tuple[torch.Tensor, int]:
    """Lay out a logical R x C matrix in row-major ('r') or column-major ('c') storage
    with leading dimension ld (>= C for row-major, >= R for column-major).
    Returns (storage tensor of shape (outer, ld), ld)."""
    R, C = logical.shape
    if layout in ("r", "row"):
        ld = C if ld is None else ld
        buf = torch.zeros((R, ld), dtype=logical.dtype)
        buf[:, :C] = logical
    else:
        ld = R if ld is None else ld
        buf = torch.zeros((C, ld), dtype=logical.dtype)
        buf[:, :R] = logical.t()
    return buf, ld


@dataclass
class Problem:
    """One GEMM+epilogue problem with its logical operands on the CPU (fp16)."""
    M: int
    N: int
    K: int
    A: torch.Tensor            # logical M x K
    B: torch.Tensor            # logical K x N
    bias: Optional[torch.Tensor]
    scale: Optional[torch.Tensor] = None
    meta: dict = field(default_factory=dict)


def make_problem(M: int, N: int, K: int, seed: int, kind: str = "uniform", bias_mode: Optional[str] = "row",
                 prologue: Optional[str] = None, ldbias: Optional[int] = None) -> Problem:
    if kind == "smallint":
        A = smallint_f16((M, K), seed * 7 + 1)
        B = smallint_f16((K, N), seed * 7 + 2)
        mk_bias = lambda shape: smallint_f16(shape, seed * 7 + 3, -8, 8)
    else:
        A = uniform_f16((M, K), seed * 7 + 1)
        B = uniform_f16((K, N), seed * 7 + 2)
        mk_bias = lambda shape: uniform_f16(shape, seed * 7 + 3)
    if bias_mode in (None, "none"):
        bias = None
    elif bias_mode == "row":
        bias = mk_bias((N,))
    elif bias_mode == "col":
        bias = mk_bias((M,))
    elif bias_mode == "full":
        ld = N if ldbias is None else ldbias
        bias = torch.zeros((M, ld), dtype=torch.float16)
        bias[:, :N] = mk_bias((M, N))
    else:
        raise ValueError(bias_mode)
    scale = None
    if prologue == "scale_k":
        scale = scale_vector(K, seed * 7 + 4, "smallint" if kind == "smallint" else "uniform")
    elif prologue == "hadamard":
        scale = hadamard_tile(M, K, seed * 7 + 5, kind)
    return Problem(M, N, K, A, B, bias, scale, {"seed": seed, "kind": kind, "bias_mode": bias_mode,
                                                "prologue": prologue})


# BASELINE.json configs (bench workloads and parity-test cases).
CONFIGS = {
    "c0_256_rr": dict(M=256, N=256, K=256, layouts=("rr",)),
    "c1_square": dict(sizes=(1024, 2048, 4096, 8192), layouts=LAYOUTS),
    "c2_deepbench_a": dict(M=5124, N=700, K=2048, layouts=("rr", "rc")),
    "c2_deepbench_b": dict(M=35, N=8457, K=2560, layouts=("rr", "rc")),
    "c3_prologue": dict(M=4096, N=4096, K=4096, layouts=("rr",), prologue="scale_k"),
    "c4_batched": dict(batch=64, M=2048, N=2048, K=2048, layouts=("rr",)),
}
