"""CPU oracle for the fused fp16 GEMM + bias + ReLU hot path (arXiv 2006.12645).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
package.  The product (``paper_2006_12645_b200``) never imports it and shares
no code with it.

The arithmetic lives in ``ge_oracle.c`` (plain fp64 triple loop, threaded over
output rows); this module only marshals numpy arrays through ctypes.  See the
header of ``ge_oracle.c`` for the definition and the paper passages it follows:
Listing 1, Listing 5 and the readings
R-C2/R-C3/R-C12 of DESIGN.md.

Functions with no pin other than the per-element bound: none -- every function
is pinned in tests/test_oracle_pins.py (codec vs numpy, golden cases, exact
rational brute force, numpy cross-check, closed forms).  Random U(-1,1) GPU
parity is judged against this oracle through the BASELINE.json bound.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from typing import Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "ge_oracle.c")
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None

LAYOUT = {"row": 0, "col": 1}
BIAS_MODE = {None: -1, "none": -1, "row": 0, "col": 1, "full": 2}
PROLOGUE = {None: 0, "none": 0, "scale_k": 1, "relu": 2, "hadamard": 3}
ACT = {None: 0, "none": 0, "relu": 1, "sigmoid": 2, "tanh": 3}


def build(force: bool = False) -> str:
    """Compile ge_oracle.c with gcc into oracle/liboracle.so (plain -O2, no fast-math)."""
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(_SRC):
        tmp = _LIB_PATH + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-fPIC", "-shared", "-std=c99", "-D_GNU_SOURCE",
                               "-fno-fast-math", "-ffp-contract=off", "-o", tmp, _SRC, "-lm", "-lpthread"])
        os.replace(tmp, _LIB_PATH)
    return _LIB_PATH


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB_PATH)
        lib.oracle_f16_to_f64.restype = ctypes.c_double
        lib.oracle_f16_to_f64.argtypes = [ctypes.c_uint16]
        lib.oracle_f64_to_f16_rne.restype = ctypes.c_uint16
        lib.oracle_f64_to_f16_rne.argtypes = [ctypes.c_double]
        P = ctypes.c_void_p
        I64 = ctypes.c_int64
        I = ctypes.c_int
        lib.oracle_f16_decode_array.argtypes = [P, P, I64]
        lib.oracle_f16_encode_array.argtypes = [P, P, I64]
        lib.oracle_gemm_epilogue.restype = I
        lib.oracle_gemm_epilogue.argtypes = [I64, I64, I64, I, I, P, I64, P, I64, P, I, I, I64, I, I, P, P, I64, I,
                                             P, I64, P, I64, P, P, I]
        lib.oracle_gemm2_epilogue.restype = I
        lib.oracle_gemm2_epilogue.argtypes = [I64, I64, I64, I64, I, I, P, I64, P, I64, P, I64, P, I64, P, I, I, I64,
                                              I, P, I64, P, I64, P, P, I]
        _lib = lib
    return _lib


def default_threads() -> int:
    return len(os.sched_getaffinity(0))


def f16_decode(bits: np.ndarray) -> np.ndarray:
    """fp16 bit patterns (uint16) -> exact fp64 values, the oracle's own decoder."""
    lib = _load()
    b = np.ascontiguousarray(bits, dtype=np.uint16)
    out = np.empty(b.shape, dtype=np.float64)
    lib.oracle_f16_decode_array(b.ctypes.data, out.ctypes.data, b.size)
    return out


def f16_encode(x: np.ndarray) -> np.ndarray:
    """fp64 -> fp16 bit patterns, round-to-nearest-even (the oracle's own encoder)."""
    lib = _load()
    v = np.ascontiguousarray(x, dtype=np.float64)
    out = np.empty(v.shape, dtype=np.uint16)
    lib.oracle_f16_encode_array(v.ctypes.data, out.ctypes.data, v.size)
    return out


def _bits(a) -> np.ndarray:
    """Accept a numpy float16/uint16 array or a CPU torch.float16 tensor; return uint16 bits."""
    if a is None:
        return None
    if hasattr(a, "numpy") and hasattr(a, "dtype") and str(a.dtype) == "torch.float16":
        import torch
        return a.detach().cpu().contiguous().view(torch.int16).numpy().view(np.uint16)
    a = np.asarray(a)
    if a.dtype == np.float16:
        return a.view(np.uint16)
    if a.dtype == np.uint16:
        return a
    raise TypeError(f"expected fp16 bits, got {a.dtype}")


def gemm_epilogue(A, B, M: int, N: int, K: int, *, layoutA: str = "row", layoutB: str = "row",
                  lda: Optional[int] = None, ldb: Optional[int] = None,
                  bias=None, bias_mode: Optional[str] = "row", ldbias: int = 0,
                  relu: bool = True, act: Optional[str] = "default", bias_sub: bool = False,
                  prologue: Optional[str] = None, scale=None, lds: Optional[int] = None,
                  literal_round: bool = False,
                  rows: Optional[Sequence[int]] = None, cols: Optional[Sequence[int]] = None,
                  nthreads: Optional[int] = None):
    """Evaluate the oracle.  Returns (out, mag) as fp64 arrays of shape (len(rows), len(cols))
    (full M x N when rows/cols are None).  A and B are fp16 storage arrays (flat or 2-D)
    read through the layout index formulas with leading dimensions lda/ldb
    (default: packed).  ``bias=None`` means no bias term.  prologue "hadamard": ``scale`` is the fp16
    storage of S (M x K in A's layout, leading dimension ``lds``, default packed).  The activation is ``act`` (None, "relu",
    "sigmoid", "tanh"); by default ReLU if ``relu`` else identity.  ``bias_sub`` subtracts the bias.
    """
    lib = _load()
    if lda is None:
        lda = K if layoutA == "row" else M
    if ldb is None:
        ldb = N if layoutB == "row" else K
    a = np.ascontiguousarray(_bits(A)).reshape(-1)
    b = np.ascontiguousarray(_bits(B)).reshape(-1)
    bm = BIAS_MODE[bias_mode] if bias is not None else -1
    bb = np.ascontiguousarray(_bits(bias)).reshape(-1) if bias is not None else None
    pro = PROLOGUE[prologue]
    sc = None
    st = None
    if pro == 3:
        st = np.ascontiguousarray(_bits(scale)).reshape(-1)
        if lds is None:
            lds = K if layoutA == "row" else M
    if pro == 1:
        sc = np.ascontiguousarray(np.asarray(scale.cpu().numpy() if hasattr(scale, "cpu") else scale,
                                             dtype=np.float32)).reshape(-1)
    r = None if rows is None else np.ascontiguousarray(np.asarray(rows, dtype=np.int64))
    c = None if cols is None else np.ascontiguousarray(np.asarray(cols, dtype=np.int64))
    nr = M if r is None else r.size
    nc = N if c is None else c.size
    out = np.empty((nr, nc), dtype=np.float64)
    mag = np.empty((nr, nc), dtype=np.float64)
    act_code = ACT["relu" if relu else None] if act == "default" else ACT[act]
    rc = lib.oracle_gemm_epilogue(
        M, N, K, LAYOUT[layoutA], LAYOUT[layoutB],
        a.ctypes.data, lda, b.ctypes.data, ldb,
        bb.ctypes.data if bb is not None else None, bm, -1 if bias_sub else 1, ldbias, act_code,
        pro, sc.ctypes.data if sc is not None else None, st.ctypes.data if st is not None else None,
        int(lds or 0), int(bool(literal_round)),
        r.ctypes.data if r is not None else None, 0 if r is None else r.size,
        c.ctypes.data if c is not None else None, 0 if c is None else c.size,
        out.ctypes.data, mag.ctypes.data, int(nthreads or default_threads()))
    if rc != 0:
        raise ValueError(f"oracle_gemm_epilogue rejected its arguments (rc={rc})")
    return out, mag


def bound(out: np.ndarray, mag: np.ndarray) -> np.ndarray:
    """BASELINE.json north_star per-element tolerance: 4e-3*mag + 1e-3*|out|."""
    return 4e-3 * mag + 1e-3 * np.abs(out)


def gemm2_epilogue(A, B, P, Q, M: int, N: int, K1: int, K2: int, *, layoutA: str = "row", layoutB: str = "row",
                   lda=None, ldb=None, ldp=None, ldq=None, bias=None, bias_mode: Optional[str] = "row",
                   ldbias: int = 0, act: Optional[str] = "relu", bias_sub: bool = False,
                   rows=None, cols=None, nthreads: Optional[int] = None):
    """Sum of matmuls (Listing 4): act(A.B + P.Q +- bias).  P, Q use the layouts of A, B."""
    lib = _load()
    lda = lda or (K1 if layoutA == "row" else M)
    ldp = ldp or (K2 if layoutA == "row" else M)
    ldb = ldb or (N if layoutB == "row" else K1)
    ldq = ldq or (N if layoutB == "row" else K2)
    arr = [np.ascontiguousarray(_bits(x)).reshape(-1) for x in (A, B, P, Q)]
    bm = BIAS_MODE[bias_mode] if bias is not None else -1
    bb = np.ascontiguousarray(_bits(bias)).reshape(-1) if bias is not None else None
    r = None if rows is None else np.ascontiguousarray(np.asarray(rows, dtype=np.int64))
    c = None if cols is None else np.ascontiguousarray(np.asarray(cols, dtype=np.int64))
    nr = M if r is None else r.size
    nc = N if c is None else c.size
    out = np.empty((nr, nc), dtype=np.float64)
    mag = np.empty((nr, nc), dtype=np.float64)
    rc = lib.oracle_gemm2_epilogue(
        M, N, K1, K2, LAYOUT[layoutA], LAYOUT[layoutB], arr[0].ctypes.data, lda, arr[1].ctypes.data, ldb,
        arr[2].ctypes.data, ldp, arr[3].ctypes.data, ldq, bb.ctypes.data if bb is not None else None, bm,
        -1 if bias_sub else 1, ldbias, ACT[act],
        r.ctypes.data if r is not None else None, 0 if r is None else r.size,
        c.ctypes.data if c is not None else None, 0 if c is None else c.size,
        out.ctypes.data, mag.ctypes.data, int(nthreads or default_threads()))
    if rc != 0:
        raise ValueError(f"oracle_gemm2_epilogue rejected its arguments (rc={rc})")
    return out, mag
