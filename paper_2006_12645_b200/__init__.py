"""paper_2006_12645_b200 -- fused fp16 GEMM + bias + ReLU for B200 (sm_100a).

Thin Python binding over the C ABI in ``include/gemm_epilogue.h`` (library
``libgemm_epilogue.so`` built in-tree by ``_build.py``).  This module only marshals
arguments (torch tensors -> pointers, strides -> leading dimensions, the current CUDA
stream); every step of the computation runs in the CUDA kernels.  There is no CPU
fallback: if the shared library is missing or the device is not sm_100 the calls raise.

Operation (Listing 1; prologue: Listing 5):
    C = epilogue(prologue(A) @ B),  epilogue = relu_add(., bias) by default.

Operands are LOGICAL matrices: ``A`` is M x K and ``B`` is K x N (optionally with a leading
batch dimension).  Each may be row-major (stride(-1) == 1) or column-major (stride(-2) == 1,
e.g. ``X.t()``); the layout pair is detected from the strides (rr, rc, cr, cc).
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional

import torch

__all__ = ["gemm_epilogue", "gemm2_epilogue", "gemm_epilogue_batched", "gemm_epilogue_host", "GEError", "plan", "validate_args",
           "launch_count", "version", "library_path", "load_library", "layout_of", "Status"]

_PKG = os.path.dirname(os.path.abspath(__file__))
# GE_DEBUG_STATS=1 selects the diagnostics build (python paper_2006_12645_b200/_build.py --debug-stats)
# (GE_LIBRARY_FILE: dev A/B experiments with an alternative in-tree build of the same library)
_LIB_PATH = os.environ.get("GE_LIBRARY_FILE") or os.path.join(
    _PKG, "libgemm_epilogue_dbg.so" if os.environ.get("GE_DEBUG_STATS") else "libgemm_epilogue.so")
_lib = None


class Status:
    OK = 0
    INVALID_VALUE = 1
    MISALIGNED = 2
    ALIASING = 3
    UNSUPPORTED_DEVICE = 4
    CUDA = 5


EPI = {"none": 0, "bias": 1, "relu": 2, "bias_relu": 3, "sigmoid": 4, "bias_sigmoid": 5, "tanh": 8, "bias_tanh": 9,
       "sub_bias": 17, "sub_bias_relu": 19, "sub_bias_sigmoid": 21, "sub_bias_tanh": 25}
EPI_F16_INTERMEDIATE = 32
BIAS_MODE = {"row": 0, "col": 1, "full": 2}
PROLOGUE = {None: 0, "none": 0, "scale_k": 1, "relu": 2, "hadamard": 3}


class GEOptions(ctypes.Structure):
    _fields_ = [("bias_mode", ctypes.c_int32), ("ldbias", ctypes.c_int64), ("prologue", ctypes.c_int32),
                ("prologue_scale", ctypes.c_void_p), ("out_dtype", ctypes.c_int32), ("tile_n", ctypes.c_int32),
                ("cta_group", ctypes.c_int32), ("stream_k", ctypes.c_int32), ("workspace", ctypes.c_void_p),
                ("workspace_bytes", ctypes.c_int64), ("multicast", ctypes.c_int32),
                ("prologue_tile", ctypes.c_void_p), ("ld_prologue_tile", ctypes.c_int64),
                ("stride_prologue_tile", ctypes.c_int64), ("tile_m", ctypes.c_int32), ("swap_ab", ctypes.c_int32)]


class GEPlanInfo(ctypes.Structure):
    _fields_ = [("tile_m", ctypes.c_int32), ("tile_n", ctypes.c_int32), ("cta_group", ctypes.c_int32),
                ("stages", ctypes.c_int32), ("num_tiles", ctypes.c_int64), ("stream_k_tiles", ctypes.c_int64),
                ("workspace_bytes", ctypes.c_int64), ("split_k", ctypes.c_int32), ("multicast", ctypes.c_int32),
                ("swap_ab", ctypes.c_int32)]


class GEError(RuntimeError):
    def __init__(self, status: int, detail: str):
        self.status = status
        super().__init__(f"{_lib.ge_status_string(status).decode()} ({detail})" if _lib else f"status {status}")


def library_path() -> str:
    return _LIB_PATH


def load_library():
    """Load libgemm_epilogue.so (built by __graft_entry__.build() / _build.py).  Raises if absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(_LIB_PATH):
        raise ImportError(f"{_LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
                          "(there is no CPU fallback)")
    lib = ctypes.CDLL(_LIB_PATH)
    I64, I32, P = ctypes.c_int64, ctypes.c_int32, ctypes.c_void_p
    OPT = ctypes.POINTER(GEOptions)
    lib.gemm_epilogue.restype = I32
    lib.gemm_epilogue.argtypes = [I64, I64, I64, I32, I32, P, I64, P, I64, P, P, I64, I32, OPT, P]
    batched = [I64, I64, I64, I64, I32, I32, P, I64, I64, P, I64, I64, P, I64, P, I64, I64, I32, OPT]
    lib.gemm_epilogue_batched.restype = I32
    lib.gemm_epilogue_batched.argtypes = batched + [P]
    lib.gemm2_epilogue.restype = I32
    lib.gemm2_epilogue.argtypes = [I64, I64, I64, I64, I32, I32, P, I64, P, I64, P, I64, P, I64, P, P, I64, I32, OPT, P]
    lib.gemm_epilogue_host.restype = I32
    lib.gemm_epilogue_host.argtypes = batched + [P]
    lib.ge_validate.restype = I32
    lib.ge_validate.argtypes = batched
    lib.ge_release_workspace.restype = I32
    lib.ge_release_workspace.argtypes = []
    lib.ge_status_string.restype = ctypes.c_char_p
    lib.ge_status_string.argtypes = [I32]
    lib.ge_last_error_detail.restype = ctypes.c_char_p
    lib.ge_last_error_detail.argtypes = []
    lib.ge_plan.restype = I32
    lib.ge_plan.argtypes = [I64, I64, I64, I64, I32, I32, OPT, I32, ctypes.POINTER(I32), ctypes.POINTER(I32),
                            ctypes.POINTER(I32), ctypes.POINTER(I32), ctypes.POINTER(I64), ctypes.POINTER(I64),
                            ctypes.POINTER(I64), ctypes.POINTER(I32)]
    lib.ge_plan_ex.restype = I32
    lib.ge_plan_ex.argtypes = [I64, I64, I64, I64, I32, I32, I32, OPT, I32, ctypes.POINTER(GEPlanInfo)]
    lib.ge_launch_count.restype = ctypes.c_uint64
    lib.ge_launch_count.argtypes = []
    lib.ge_debug_read.restype = I32
    lib.ge_debug_read.argtypes = [P, I32]
    lib.ge_version.restype = ctypes.c_char_p
    lib.ge_version.argtypes = []
    lib.ge_tensor_map_cache_stats.restype = None
    lib.ge_tensor_map_cache_stats.argtypes = [ctypes.POINTER(ctypes.c_uint64), ctypes.POINTER(ctypes.c_uint64)]
    _lib = lib
    return lib


def _check(status: int):
    if status != Status.OK:
        raise GEError(status, _lib.ge_last_error_detail().decode())


def layout_of(x: torch.Tensor):
    """(layout, ld) of the last two dims of a logical matrix view: 0 = row-major, 1 = col-major."""
    R, C = x.shape[-2], x.shape[-1]
    s0, s1 = x.stride(-2), x.stride(-1)
    up8 = lambda v: (max(v, 1) + 7) // 8 * 8     # a single row/column: any ld >= extent is valid
    if C == 1 and s0 == 1 and R > 1:
        return 1, up8(R)
    if (s1 == 1 or C <= 1) and (R <= 1 or s0 >= C):
        return 0, (s0 if R > 1 else up8(C))
    if (s0 == 1 or R <= 1) and (C <= 1 or s1 >= R):
        return 1, (s1 if C > 1 else up8(R))
    raise ValueError(f"operand with shape {tuple(x.shape)} and strides {x.stride()} is neither row- nor column-major")


_workspaces = {}


def _workspace(device, stream_handle):
    """Zero-filled stream-K / split-K workspace for (device, stream), large enough for any plan
    (one fp32 128 x 256 slot, one flag and one tile counter per SM).  Allocated through torch, so it is CUDA-graph safe; every
    launch leaves it zero-filled."""
    key = (device.index if hasattr(device, "index") else int(device), int(stream_handle))
    ws = _workspaces.get(key)
    if ws is None and torch.cuda.is_current_stream_capturing():
        # allocating here would capture its zero-fill into the graph (replayed every time): no
        # workspace, so the library plans without stream-K (split-K needs none)
        return None
    if ws is None:
        sms = torch.cuda.get_device_properties(device).multi_processor_count
        ws = torch.zeros(sms * (128 * 256 * 4 + 8), dtype=torch.uint8, device=device)
        _workspaces[key] = ws
    return ws


def clear_workspaces():
    _workspaces.clear()


_opt_cache = {}


def _options(bias_mode, ldbias, prologue, scale, out_dtype, tile_n, cta_group, stream_k=0, ws=None, multicast=0,
             tile=None, swap_ab=0, tile_m=0):
    """ge_options for these arguments; reused across calls with the same ones (per-call host cost).
    tile: (ptr, ld, batch stride) of the Hadamard prologue operand S."""
    key = (bias_mode, ldbias, prologue, scale.data_ptr() if scale is not None else 0, out_dtype, tile_n,
           cta_group, stream_k, ws.data_ptr() if ws is not None else 0, ws.numel() if ws is not None else 0,
           multicast, tile, swap_ab, tile_m)
    o = _opt_cache.get(key)
    if o is not None:
        return o
    o = GEOptions()
    o.stream_k = int(stream_k)
    o.workspace = ws.data_ptr() if ws is not None else None
    o.workspace_bytes = ws.numel() if ws is not None else 0
    o.bias_mode = BIAS_MODE[bias_mode]
    o.ldbias = int(ldbias or 0)
    o.prologue = PROLOGUE[prologue]
    o.prologue_scale = scale.data_ptr() if (scale is not None and prologue == "scale_k") else None
    if tile is not None:
        o.prologue_tile, o.ld_prologue_tile, o.stride_prologue_tile = tile
    o.out_dtype = 1 if out_dtype == torch.float32 else 0
    o.tile_n = int(tile_n)
    o.cta_group = int(cta_group)
    o.multicast = int(multicast)
    o.swap_ab = int(swap_ab)
    o.tile_m = int(tile_m)
    if len(_opt_cache) > 512:
        _opt_cache.clear()
    _opt_cache[key] = o
    return o


def _prologue_tile(prologue, scale, A, batch=None):
    """(ptr, ld, batch stride) of the Hadamard operand S (prologue="hadamard", passed as `scale`):
    fp16, the logical shape of A ((M, K), or (batch, M, K) / a shared (M, K) for batched calls),
    stored in A's layout (DESIGN.md R-C18)."""
    if prologue != "hadamard":
        return None
    if scale is None:
        raise ValueError("prologue 'hadamard' needs scale = the (M, K) fp16 tile S")
    if scale.dtype != torch.float16:
        raise ValueError(f"the Hadamard tile must be float16, got {scale.dtype}")
    if scale.shape[-2:] != A.shape[-2:] or scale.dim() not in ((2, 3) if batch is not None else (2,)):
        raise ValueError(f"the Hadamard tile must have A's shape {tuple(A.shape[-2:])}, got {tuple(scale.shape)}")
    if scale.dim() == 3 and scale.shape[0] != batch:
        raise ValueError("per-item Hadamard tiles need one per batch item")
    if scale.device != A.device:
        raise ValueError("the Hadamard tile must be on A's device")
    ls, lds = layout_of(scale)
    la, _ = layout_of(A)
    if ls != la:
        raise ValueError("the Hadamard tile must have A's layout (row- or column-major)")
    return (scale.data_ptr(), lds, scale.stride(0) if scale.dim() == 3 else 0)


def _stream(stream, device_index: Optional[int] = None) -> int:
    if stream is None:
        if device_index is None:
            device_index = torch.cuda.current_device()
        return torch._C._cuda_getCurrentRawStream(device_index)
    return stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)


def _op(op: str, bias) -> int:
    """op name -> ge_epilogue_op flags; a "literal_" prefix (e.g. "literal_bias_relu") selects the
    paper-literal rounding point act(fp16(fp16(acc) +- bias)) (GE_EPI_F16_INTERMEDIATE, DESIGN.md R-C3)."""
    if op is None:
        op = "bias_relu" if bias is not None else "relu"
    if op.startswith("literal_"):
        return EPI[op[len("literal_"):]] | EPI_F16_INTERMEDIATE
    return EPI[op]


def _check_tensors(M, N, K, *, ops, bias=None, bias_mode="row", scale=None, out=None, batch=None, host=False):
    """Argument checks the C ABI cannot make (it sees raw pointers): dtypes, shapes against M/N/K
    and the bias mode, and that every tensor lives on one CUDA device (or on the host for the
    host-buffer entry).  Raises ValueError; nothing is launched."""
    dev = None
    def where(name, t):
        nonlocal dev
        if host:
            if t.is_cuda:
                raise ValueError(f"{name} must be a host (CPU) tensor for gemm_epilogue_host")
            return
        if not t.is_cuda:
            raise ValueError(f"{name} must be a CUDA tensor")
        if dev is None:
            dev = t.device
        elif t.device != dev:
            raise ValueError(f"{name} is on {t.device}, expected {dev}")
    for name, t in ops:
        if t.dtype != torch.float16:
            raise ValueError(f"{name} must be float16, got {t.dtype}")
        where(name, t)
    lead = () if batch is None else (batch,)
    if bias is not None:
        if bias.dtype != torch.float16:
            raise ValueError(f"bias must be float16, got {bias.dtype}")
        where("bias", bias)
        if bias_mode not in BIAS_MODE:
            raise ValueError(f"bias_mode must be one of {sorted(BIAS_MODE)}")
        if bias_mode == "full":
            ok = bias.dim() in ((2, 3) if batch is not None else (2,)) and bias.shape[-2] == M and bias.shape[-1] >= N
            if ok and bias.dim() == 3:
                ok = bias.shape[0] == batch
            if not ok:
                raise ValueError(f"full bias must be (M, >=N){' or (batch, M, >=N)' if batch is not None else ''}, "
                                 f"got {tuple(bias.shape)}")
        else:
            L = N if bias_mode == "row" else M
            ok = (bias.dim() == 1 and bias.shape[0] == L) or \
                 (batch is not None and bias.dim() == 2 and tuple(bias.shape) == (batch, L))
            if not ok:
                raise ValueError(f"{bias_mode} bias must have length {'N' if bias_mode == 'row' else 'M'} = {L}"
                                 f"{' (or shape (batch, ' + str(L) + '))' if batch is not None else ''}, got "
                                 f"{tuple(bias.shape)}")
    if scale is not None:
        if scale.dtype != torch.float32:
            raise ValueError(f"scale must be float32, got {scale.dtype}")
        if scale.dim() != 1 or scale.numel() < K or scale.stride(0) != 1:
            raise ValueError(f"scale must be a contiguous 1-D tensor of length >= K = {K}")
        where("scale", scale)
    if out is not None:
        if out.dtype not in (torch.float16, torch.float32):
            raise ValueError(f"out must be float16 or float32, got {out.dtype}")
        if tuple(out.shape) != lead + (M, N):
            raise ValueError(f"out must have shape {lead + (M, N)}, got {tuple(out.shape)}")
        where("out", out)


def _bias_ld(bias, bias_mode):
    if bias is None:
        return 0, 0
    if bias_mode == "full":
        if bias.stride(-1) != 1:
            raise ValueError("FULL bias must be row-major (stride(-1) == 1)")
        return bias.stride(-2), (bias.stride(0) if bias.dim() == 3 else 0)
    if bias.stride(-1) != 1:
        raise ValueError("bias vector must be contiguous")
    return 0, (bias.stride(0) if bias.dim() == 2 else 0)


def gemm_epilogue(A: torch.Tensor, B: torch.Tensor, bias: Optional[torch.Tensor] = None, *, op: Optional[str] = None,
                  bias_mode: str = "row", prologue: Optional[str] = None, scale: Optional[torch.Tensor] = None,
                  out_dtype: torch.dtype = torch.float16, out: Optional[torch.Tensor] = None, tile_n: int = 0,
                  cta_group: int = 0, stream_k: int = 0, multicast: int = 0, swap_ab: int = 0,
                  tile_m: int = 0, stream=None) -> torch.Tensor:
    """C = relu_add(prologue(A) @ B, bias) on the current CUDA device (fp16 in, fp32 accumulate).

    A: (M, K) fp16, B: (K, N) fp16, row- or column-major views.  bias: (N,) for bias_mode "row",
    (M,) for "col", (M, ldbias>=N) row-major for "full".  op in {"none", "bias", "relu", "bias_relu",
    "sigmoid", "bias_sigmoid", "tanh", "bias_tanh", "sub_bias", "sub_bias_relu", "sub_bias_sigmoid",
    "sub_bias_tanh"}, each optionally prefixed "literal_" for the paper-literal fp16 rounding of the
    intermediate (default: bias_relu if bias is given else relu).  prologue "scale_k" (scale: (K,) fp32),
    "relu", or "hadamard" (scale: the (M, K) fp16 tile S in A's layout, a'(i,k) = fp16(S[i,k] * A[i,k])).
    Returns C (M, N) row-major in out_dtype (fp16 or fp32), asynchronously on the current stream.
    """
    lib = load_library()
    if A.dim() != 2 or B.dim() != 2:
        raise ValueError("use gemm_epilogue_batched for 3-D operands")
    M, K = A.shape
    K2, N = B.shape
    if K2 != K:
        raise ValueError(f"inner dimensions differ: A is {tuple(A.shape)}, B is {tuple(B.shape)}")
    if prologue == "scale_k" and scale is None:
        raise ValueError("prologue 'scale_k' needs scale")
    tile = _prologue_tile(prologue, scale, A)
    _check_tensors(M, N, K, ops=(("A", A), ("B", B)), bias=bias, bias_mode=bias_mode,
                   scale=scale if prologue == "scale_k" else None, out=out)
    la, lda = layout_of(A)
    lb, ldb = layout_of(B)
    if out is None:
        out = torch.empty((M, N), dtype=out_dtype, device=A.device)
    if out.stride(-1) != 1 and N > 1:
        raise ValueError("out must be row-major")
    ldbias, _ = _bias_ld(bias, bias_mode)
    sh = _stream(stream, A.get_device())
    o = _options(bias_mode, ldbias, prologue, scale, out.dtype, tile_n, cta_group, stream_k,
                 _workspace(A.device, sh) if stream_k != 1 else None, multicast, tile, swap_ab, tile_m)
    st = lib.gemm_epilogue(M, N, K, la, lb, A.data_ptr(), lda, B.data_ptr(), ldb,
                           bias.data_ptr() if bias is not None else None, out.data_ptr(), max(out.stride(0), N, 1),
                           _op(op, bias), ctypes.byref(o), sh)
    _check(st)
    return out


def gemm2_epilogue(A: torch.Tensor, B: torch.Tensor, P: torch.Tensor, Q: torch.Tensor,
                   bias: Optional[torch.Tensor] = None, *, op: Optional[str] = None, bias_mode: str = "row",
                   out_dtype: torch.dtype = torch.float16, out: Optional[torch.Tensor] = None, tile_n: int = 0,
                   cta_group: int = 0, stream_k: int = 0, multicast: int = 0, swap_ab: int = 0,
                  tile_m: int = 0, stream=None) -> torch.Tensor:
    """Sum of matmuls (Listing 4): C = epilogue(A @ B + P @ Q) in one kernel, one TMEM
    accumulator.  A (M, K1), B (K1, N), P (M, K2), Q (K2, N); P must share A's layout (row/col
    major) and Q B's."""
    lib = load_library()
    M, K1 = A.shape
    N = B.shape[1]
    K2 = P.shape[1]
    if B.shape[0] != K1 or P.shape[0] != M or Q.shape != (K2, N):
        raise ValueError("shapes of A.B and P.Q disagree")
    _check_tensors(M, N, K1, ops=(("A", A), ("B", B), ("P", P), ("Q", Q)), bias=bias, bias_mode=bias_mode, out=out)
    la, lda = layout_of(A)
    lb, ldb = layout_of(B)
    lp, ldp = layout_of(P)
    lq, ldq = layout_of(Q)
    if lp != la or lq != lb:
        raise ValueError("P must have A's layout and Q must have B's layout")
    if out is None:
        out = torch.empty((M, N), dtype=out_dtype, device=A.device)
    if out.stride(-1) != 1 and N > 1:
        raise ValueError("out must be row-major")
    ldbias, _ = _bias_ld(bias, bias_mode)
    sh = _stream(stream, A.get_device())
    o = _options(bias_mode, ldbias, None, None, out.dtype, tile_n, cta_group, stream_k,
                 _workspace(A.device, sh) if stream_k != 1 else None, multicast, None, swap_ab, tile_m)
    st = lib.gemm2_epilogue(M, N, K1, K2, la, lb, A.data_ptr(), lda, B.data_ptr(), ldb, P.data_ptr(), ldp,
                            Q.data_ptr(), ldq, bias.data_ptr() if bias is not None else None, out.data_ptr(),
                            max(out.stride(0), N, 1), _op(op, bias), ctypes.byref(o), sh)
    _check(st)
    return out


def _batched_args(A, B, bias, bias_mode, out, scale=None, host=False):
    if A.dim() != 3 or B.dim() != 3:
        raise ValueError("batched operands are (batch, rows, cols)")
    batch, M, K = A.shape
    _, K2, N = B.shape
    if K2 != K or B.shape[0] != batch:
        raise ValueError("batched shapes disagree")
    _check_tensors(M, N, K, ops=(("A", A), ("B", B)), bias=bias, bias_mode=bias_mode, scale=scale,
                   out=(out if out is None or out.dim() == 3 else out.unsqueeze(0)), batch=batch, host=host)
    if out is not None and out.stride(-1) != 1 and N > 1:
        raise ValueError("out must be row-major")
    la, lda = layout_of(A)
    lb, ldb = layout_of(B)
    ldbias, sbias = _bias_ld(bias, bias_mode)
    return batch, M, N, K, la, lda, A.stride(0), lb, ldb, B.stride(0), ldbias, sbias


def gemm_epilogue_batched(A: torch.Tensor, B: torch.Tensor, bias: Optional[torch.Tensor] = None, *,
                          op: Optional[str] = None, bias_mode: str = "row", prologue: Optional[str] = None,
                          scale: Optional[torch.Tensor] = None, out_dtype: torch.dtype = torch.float16,
                          out: Optional[torch.Tensor] = None, tile_n: int = 0, cta_group: int = 0,
                          stream_k: int = 0, multicast: int = 0, swap_ab: int = 0, tile_m: int = 0,
                          stream=None) -> torch.Tensor:
    """Strided-batched form: A (b, M, K), B (b, K, N), bias (N,)/(b, N) [row], (M,)/(b, M) [col],
    (M, ld)/(b, M, ld) [full]; a 1-D/2-D bias is shared by every item.  One persistent launch."""
    lib = load_library()
    if prologue == "scale_k" and scale is None:
        raise ValueError("prologue 'scale_k' needs scale")
    batch, M, N, K, la, lda, sA, lb, ldb, sB, ldbias, sbias = _batched_args(
        A, B, bias, bias_mode, out, scale if prologue == "scale_k" else None)
    tile = _prologue_tile(prologue, scale, A, batch)
    if out is None:
        out = torch.empty((batch, M, N), dtype=out_dtype, device=A.device)
    sh = _stream(stream, A.get_device())
    o = _options(bias_mode, ldbias, prologue, scale, out.dtype, tile_n, cta_group, stream_k,
                 _workspace(A.device, sh) if stream_k != 1 else None, multicast, tile, swap_ab, tile_m)
    st = lib.gemm_epilogue_batched(batch, M, N, K, la, lb, A.data_ptr(), lda, sA, B.data_ptr(), ldb, sB,
                                   bias.data_ptr() if bias is not None else None, sbias, out.data_ptr(),
                                   max(out.stride(1), N, 1), out.stride(0), _op(op, bias), ctypes.byref(o), sh)
    _check(st)
    return out


def gemm_epilogue_host(A: torch.Tensor, B: torch.Tensor, bias: Optional[torch.Tensor] = None, *,
                       op: Optional[str] = None, bias_mode: str = "row", prologue: Optional[str] = None,
                       scale: Optional[torch.Tensor] = None, out: Optional[torch.Tensor] = None,
                       out_dtype: torch.dtype = torch.float16, tile_n: int = 0, cta_group: int = 0,
                       stream_k: int = 0, multicast: int = 0, swap_ab: int = 0, tile_m: int = 0,
                          stream=None) -> torch.Tensor:
    """End-to-end path through the C ABI with HOST (CPU, ideally pinned) tensors: the library copies
    the inputs to the device, runs the fused kernel and copies C back, synchronously."""
    lib = load_library()
    A3 = A if A.dim() == 3 else A.unsqueeze(0)
    B3 = B if B.dim() == 3 else B.unsqueeze(0)
    if prologue == "scale_k" and scale is None:
        raise ValueError("prologue 'scale_k' needs scale")
    out3 = None if out is None else (out if out.dim() == 3 else out.unsqueeze(0))
    batch, M, N, K, la, lda, sA, lb, ldb, sB, ldbias, sbias = _batched_args(
        A3, B3, bias, bias_mode, out3, scale if prologue == "scale_k" else None, host=True)
    tile = _prologue_tile(prologue, scale, A3, batch)
    if out is None:
        out = torch.empty((batch, M, N) if A.dim() == 3 else (M, N), dtype=out_dtype,
                          pin_memory=A.is_pinned())
    out3 = out if out.dim() == 3 else out.unsqueeze(0)
    o = _options(bias_mode, ldbias, prologue, scale, out.dtype, tile_n, cta_group, stream_k, multicast=multicast,
                 tile=tile, swap_ab=swap_ab, tile_m=tile_m)
    st = lib.gemm_epilogue_host(batch, M, N, K, la, lb, A3.data_ptr(), lda, sA, B3.data_ptr(), ldb, sB,
                                bias.data_ptr() if bias is not None else None, sbias, out3.data_ptr(),
                                max(out3.stride(1), N, 1), out3.stride(0), _op(op, bias), ctypes.byref(o),
                                _stream(stream))
    _check(st)
    return out


def validate_args(*args) -> int:
    """Raw ge_validate (19 arguments, see include/gemm_epilogue.h); returns the status code."""
    return load_library().ge_validate(*args)


def plan(M: int, N: int, K: int, batch: int = 1, layouts: str = "rr", num_sms: int = 148, tile_n: int = 0,
         cta_group: int = 0, stream_k: int = 0, prologue: Optional[str] = None, multicast: int = 0,
         swap_ab: int = 0, op: str = "bias_relu", bias_mode: str = "row", tile_m: int = 0) -> dict:
    """The launch configuration the library's planner picks (ge_plan_ex), assuming a stream-K
    workspace is passed (the device entry points of this binding always pass one)."""
    lib = load_library()
    o = _options(bias_mode, 0, prologue, None, torch.float16, tile_n, cta_group, stream_k, multicast=multicast,
                 swap_ab=swap_ab, tile_m=tile_m)
    info = GEPlanInfo()
    st = lib.ge_plan_ex(batch, M, N, K, 0 if layouts[0] == "r" else 1, 0 if layouts[1] == "r" else 1,
                        _op(op, True), ctypes.byref(o), num_sms, ctypes.byref(info))
    _check(st)
    return {f: getattr(info, f) for f, _ in GEPlanInfo._fields_}


def launch_count() -> int:
    return int(load_library().ge_launch_count())


def tensor_map_cache_stats() -> dict:
    """{"hits": maps reused, "misses": maps encoded} of the library's tensor-map cache."""
    h, m = ctypes.c_uint64(), ctypes.c_uint64()
    load_library().ge_tensor_map_cache_stats(ctypes.byref(h), ctypes.byref(m))
    return {"hits": h.value, "misses": m.value}


def debug_stats(max_ctas: int = 148):
    """Per-CTA blocked-cycle counters of the last launch (needs GE_DEBUG_STATS=1), as a list of
    dicts, or [] when diagnostics are off.  Synchronizes."""
    import numpy as np
    buf = np.zeros((max_ctas, 30), dtype=np.uint64)
    n = load_library().ge_debug_read(buf.ctypes.data, max_ctas)
    keys = ("total", "prod_wait_empty", "mma_wait_full", "mma_wait_tempty", "epi_wait_tfull", "epi_to_release0",
            "epi_to_release1", "epi_tile", "epi_tmem_ld", "epi_math", "sk_owner_wait", "sk_partial_write",
            "sk_pieces", "epi_end", "reserved", "first_mma", "g_entry", "g_start", "g_epi_end", "g_exit",
            "xf_wait", "xf_work", "mma_issue", "mma_commit", "prod_issue", "prod_total",
            "own_ld", "own_add", "own_math", "own_st")
    return [dict(zip(keys, (int(x) for x in buf[i, :30]))) for i in range(n)]


def version() -> str:
    return load_library().ge_version().decode()
