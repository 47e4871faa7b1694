"""CPU-side tests of the C ABI library: it builds, loads, exports every symbol that
include/gemm_epilogue.h declares, validates arguments exactly as documented, plans tiles, and
fails loudly (no CPU fallback) when there is no sm_100 device.  No kernel is launched here."""
from __future__ import annotations

import ctypes
import os
import re

import pytest
import torch

from paper_2006_12645_b200 import _build

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "gemm_epilogue.h")


@pytest.fixture(scope="module")
def ge():
    _build.build()
    import paper_2006_12645_b200 as ge
    ge.load_library()
    return ge


@pytest.fixture(scope="module")
def lib(ge):
    return ge.load_library()


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(?:ge_status|uint64_t|int32_t|void|const char\*)\s+(\w+)\s*\(", src)))


def test_exports_every_declared_symbol(lib):
    names = declared_functions()
    assert {"gemm_epilogue", "gemm_epilogue_batched", "gemm_epilogue_host", "ge_validate", "ge_status_string",
            "ge_last_error_detail", "ge_plan", "ge_launch_count", "ge_version",
            "ge_release_workspace", "ge_debug_read", "ge_tensor_map_cache_stats"} <= set(names)
    for n in names:
        assert hasattr(lib, n), n


def test_library_is_sm100a_native(lib):
    """The .so carries sm_100a SASS with tcgen05 MMA, TMEM loads and TMA (B200_PROFILING.md table)."""
    import shutil
    import subprocess
    exe = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(exe):
        pytest.skip("cuobjdump not available")
    out = subprocess.run([exe, "-sass", _build.LIB], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    for mnem in ("UTCHMMA", "LDTM", "UTMALDG", "UTMASTG"):
        assert mnem in out, mnem
    assert "HMMA.16816" not in out          # no legacy mma.sync path


def test_strings(lib):
    for s in range(6):
        assert lib.ge_status_string(s).startswith(b"GE_")
    assert lib.ge_status_string(99) == b"unknown ge_status"
    assert b"sm_100a" in lib.ge_version()


# ------------------------------------------------------------------ validation matrix
P = 0x10000          # fake, 16-byte aligned, never dereferenced (ge_validate only compares pointers)


def v(lib, batch=1, M=128, N=128, K=64, la=0, lb=0, A=P, lda=0, sA=0, B=P * 16, ldb=0, sB=0, bias=P * 64, sBias=0,
      C=P * 128, ldc=0, sC=0, op=3, opt=None):
    return lib.ge_validate(batch, M, N, K, la, lb, A, lda, sA, B, ldb, sB, bias, sBias, C, ldc, sC, op,
                           ctypes.byref(opt) if opt is not None else None)


def opts(ge, **kw):
    o = ge.GEOptions()
    o.bias_mode, o.ldbias, o.prologue, o.prologue_scale, o.out_dtype, o.tile_n, o.cta_group = 0, 0, 0, None, 0, 0, 0
    o.stream_k, o.workspace, o.workspace_bytes = 0, None, 0
    for k, val in kw.items():
        setattr(o, k, val)
    return o


def test_validate_ok(lib, ge):
    assert v(lib) == 0
    for la in (0, 1):
        for lb in (0, 1):
            assert v(lib, la=la, lb=lb) == 0
    assert v(lib, M=0) == 0 and v(lib, N=0) == 0 and v(lib, batch=0) == 0      # no-ops
    assert v(lib, K=0, A=0, B=0) == 0                                           # K = 0: A/B unused


def test_validate_invalid_values(lib, ge):
    S = ge.Status
    assert v(lib, M=-1) == S.INVALID_VALUE
    assert v(lib, K=-5) == S.INVALID_VALUE
    assert v(lib, batch=-1) == S.INVALID_VALUE
    assert v(lib, M=1 << 31) == S.INVALID_VALUE
    assert v(lib, la=2) == S.INVALID_VALUE
    assert v(lib, op=6) == S.INVALID_VALUE             # two activations
    assert v(lib, op=16) == S.INVALID_VALUE            # subtract without a bias
    assert v(lib, op=64) == S.INVALID_VALUE
    assert v(lib, op=32 | 3) == 0 and v(lib, op=32 | 2) == 0   # paper-literal rounding modifier (R-C3)
    assert v(lib, op=32 | 6) == S.INVALID_VALUE
    assert v(lib, op=4) == 0 and v(lib, op=9) == 0 and v(lib, op=25) == 0
    assert v(lib, lda=32) == S.INVALID_VALUE            # row-major A needs lda >= K = 64
    assert v(lib, la=1, lda=64) == S.INVALID_VALUE      # col-major A needs lda >= M = 128
    assert v(lib, ldb=64) == S.INVALID_VALUE            # row-major B needs ldb >= N
    assert v(lib, ldc=100) == S.INVALID_VALUE
    assert v(lib, C=0) == S.INVALID_VALUE
    assert v(lib, A=0) == S.INVALID_VALUE
    assert v(lib, bias=0) == S.INVALID_VALUE            # op has a bias
    assert v(lib, bias=0, op=2) == 0                    # relu only: no bias needed
    assert v(lib, opt=opts(ge, bias_mode=3)) == S.INVALID_VALUE
    assert v(lib, opt=opts(ge, prologue=1)) == S.INVALID_VALUE          # SCALE_K without a scale
    assert v(lib, opt=opts(ge, prologue=1, prologue_scale=P * 512)) == 0
    assert v(lib, opt=opts(ge, out_dtype=2)) == S.INVALID_VALUE
    assert v(lib, opt=opts(ge, tile_n=96)) == S.INVALID_VALUE
    assert v(lib, opt=opts(ge, cta_group=3)) == S.INVALID_VALUE
    assert v(lib, opt=opts(ge, cta_group=2, tile_n=64)) == S.INVALID_VALUE
    assert v(lib, opt=opts(ge, cta_group=1, tile_n=192)) == 0
    assert v(lib, lb=1, opt=opts(ge, cta_group=2, tile_n=192)) == 0                # K-major B
    assert v(lib, lb=0, opt=opts(ge, cta_group=2, tile_n=192)) == S.INVALID_VALUE  # pair 192 needs K-major B
    assert v(lib, opt=opts(ge, bias_mode=2, ldbias=64)) == S.INVALID_VALUE   # ldbias < N
    assert v(lib, batch=2, sC=100) == S.INVALID_VALUE   # output items would overlap
    assert v(lib, opt=opts(ge, stream_k=3)) == S.INVALID_VALUE
    assert v(lib, opt=opts(ge, workspace=P + 4, workspace_bytes=1 << 20)) == S.INVALID_VALUE   # misaligned
    assert lib.ge_last_error_detail()                    # a reason is recorded
    assert v(lib, opt=opts(ge, workspace=P * 1024, workspace_bytes=1 << 20)) == 0


def test_validate_alignment(lib, ge):
    S = ge.Status
    assert v(lib, A=P + 2) == S.MISALIGNED
    assert v(lib, B=P * 16 + 8) == S.MISALIGNED
    assert v(lib, K=60, lda=60) == S.MISALIGNED          # 120-byte rows break the TMA stride rule
    assert v(lib, batch=2, sA=128 * 64 + 4) == S.MISALIGNED
    assert v(lib, C=P * 128 + 2) == 0                    # C/bias have a st.global fallback
    assert v(lib, N=37, ldc=37, ldb=40) == 0


def test_validate_aliasing(lib, ge):
    S = ge.Status
    assert v(lib, C=P) == S.ALIASING                     # C == A
    assert v(lib, C=P * 16 + 64) == S.ALIASING           # C inside B
    assert v(lib, C=P * 64) == S.ALIASING                # C == bias
    assert v(lib, C=P * 64 - 2 * 128 * 128 + 2) == S.ALIASING   # C's tail overlaps bias


def test_plan_tiles(ge):
    p = ge.plan(8192, 8192, 8192, tile_n=256, cta_group=1)
    assert p["tile_m"] == 128 and p["tile_n"] == 256 and p["num_tiles"] == 64 * 32
    p = ge.plan(8192, 8192, 8192, tile_n=256, cta_group=2)
    assert p["tile_m"] == 256 and p["num_tiles"] == 32 * 32
    p = ge.plan(35, 8457, 2560)                        # skinny M: swap-AB, N = 8457 on the 128-row MMA side
    assert p["swap_ab"] == 1 and (p["tile_n"], p["cta_group"]) == (64, 1) and p["num_tiles"] == 67
    p = ge.plan(35, 8457, 2560, swap_ab=1)             # unswapped: 128 x 128 tiles over the 8457 columns
    assert p["swap_ab"] == 0 and (p["tile_n"], p["cta_group"]) == (128, 1) and p["num_tiles"] == 67
    assert ge.plan(35, 8457, 2560, prologue="scale_k")["swap_ab"] == 0           # prologue on A: no swap
    assert ge.plan(35, 8457, 2560, bias_mode="full")["swap_ab"] == 0             # FULL bias: no swap
    assert ge.plan(300, 520, 200, swap_ab=2)["swap_ab"] == 1                     # forced where legal
    p = ge.plan(1024, 1024, 1024)                      # small: narrow tiles to fill the SMs
    assert p["tile_n"] == 64 and p["num_tiles"] == 128
    p = ge.plan(2048, 2048, 2048, batch=64)           # large: the 256 x 256 CTA-pair tile
    assert p["cta_group"] == 2 and p["tile_n"] == 256 and p["num_tiles"] == 64 * 8 * 8
    assert p["stages"] >= 4
    p = ge.plan(8192, 8192, 8192)
    assert p["cta_group"] == 2 and p["tile_n"] in (256, 512)
    # stream-K: only the last partial wave is split; workspace = one fp32 128 x BN slot + flag per CTA
    p = ge.plan(4096, 4096, 4096, tile_n=256, cta_group=2, stream_k=2)
    assert p["num_tiles"] == 256 and p["stream_k_tiles"] == 256 % 74
    assert p["workspace_bytes"] == 148 * (128 * 256 * 4 + 4)
    assert ge.plan(4096, 4096, 4096, tile_n=256, cta_group=2, stream_k=1)["stream_k_tiles"] == 0
    assert ge.plan(8192, 8192, 8192, tile_n=512, cta_group=2, stream_k=2)["stream_k_tiles"] == 0   # 1-buffer acc
    # split-K: few long tiles -> clusters of S single-CTA tiles reducing in DSMEM (no workspace)
    p = ge.plan(2048, 128, 3456, layouts="rc")
    assert p["cta_group"] == 1 and 2 <= p["split_k"] <= 8 and p["workspace_bytes"] == 0
    assert p["num_tiles"] * p["split_k"] <= 148
    assert ge.plan(2048, 128, 3456, layouts="rc", stream_k=1)["split_k"] == 1               # off
    assert ge.plan(8192, 8192, 8192)["split_k"] == 1
    assert ge.plan(2048, 128, 3456, layouts="rc", cta_group=2)["split_k"] == 1             # pairs never split
    with pytest.raises(ge.GEError):
        ge.plan(8192, 8192, 8192, tile_n=96)


def test_no_device_fails_loudly(ge):
    """Without an sm_100 device the product raises; it never computes on the CPU."""
    if torch.cuda.is_available():
        pytest.skip("has a GPU")
    A = torch.zeros((64, 64), dtype=torch.float16)
    with pytest.raises(Exception):
        ge.gemm_epilogue(A, A)


def test_missing_library_fails_loudly(tmp_path):
    """Without the compiled CUDA library the package raises on first use (ImportError naming the
    build command); there is no CPU fallback path to take instead."""
    import subprocess
    import sys
    code = ("import torch, paper_2006_12645_b200 as ge\n"
            "try:\n"
            "    ge.gemm_epilogue(torch.zeros((8, 8), dtype=torch.float16), torch.zeros((8, 8), dtype=torch.float16))\n"
            "except ImportError as e:\n"
            "    print('IMPORTERROR', e)\n")
    env = dict(os.environ, GE_LIBRARY_FILE=str(tmp_path / "absent.so"))
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env,
                       cwd=os.path.dirname(os.path.dirname(os.path.abspath(__file__))), timeout=300)
    assert "IMPORTERROR" in r.stdout and "build" in r.stdout, (r.stdout, r.stderr[-500:])


def test_binding_layout_detection(ge):
    X = torch.zeros((96, 40), dtype=torch.float16)
    assert ge.layout_of(X) == (0, 40)
    assert ge.layout_of(X.t()) == (1, 40)
    Y = torch.zeros((96, 48), dtype=torch.float16)[:, :40]
    assert ge.layout_of(Y) == (0, 48)
    with pytest.raises(ValueError):
        ge.layout_of(torch.zeros((8, 8, 2), dtype=torch.float16)[:, :, 0])


def test_plan_rejects_what_launch_rejects(ge):
    """ge_plan runs the launch entry points' option checks: invalid combinations are
    GE_ERR_INVALID_VALUE instead of an arbitrary plan."""
    for kw in (dict(multicast=2, tile_n=64), dict(multicast=2, prologue="scale_k"), dict(multicast=3),
               dict(tile_n=192, cta_group=2, layouts="rr"), dict(tile_n=512, cta_group=1), dict(cta_group=3),
               dict(stream_k=3)):
        with pytest.raises(ge.GEError) as e:
            ge.plan(1024, 1024, 1024, **kw)
        assert e.value.status == ge.Status.INVALID_VALUE, kw
    assert ge.plan(1024, 1024, 1024, tile_n=192, cta_group=2, layouts="rc")["tile_n"] == 192


def test_binding_rejects_bad_tensors(ge):
    """The binding checks what the C ABI cannot see (dtype, shape, device) before any launch
    (ADVICE r1): wrong dtypes, an output of the wrong shape, a bias of the wrong length for its
    mode, a short or non-fp32 scale, and device tensors for the host entry all raise ValueError."""
    h = lambda *s: torch.zeros(s, dtype=torch.float16)
    A, B, bias = h(64, 32), h(32, 48), h(48)
    bad = [
        dict(A=A.float()), dict(B=B.to(torch.bfloat16)), dict(bias=bias.float()), dict(bias=h(47)),
        dict(bias=h(64), bias_mode="row"), dict(bias=h(48), bias_mode="col"), dict(bias=h(64, 40), bias_mode="full"),
        dict(out=torch.zeros((64, 47), dtype=torch.float16)), dict(out=torch.zeros((64, 48), dtype=torch.bfloat16)),
        dict(prologue="scale_k", scale=torch.ones(31)), dict(prologue="scale_k", scale=torch.ones(32).double()),
        dict(prologue="scale_k", scale=None),
    ]
    for kw in bad:
        args = dict(A=A, B=B, bias=bias)
        args.update(kw)
        with pytest.raises(ValueError):
            ge.gemm_epilogue_host(args.pop("A"), args.pop("B"), args.pop("bias"), **args)
    with pytest.raises(ValueError):                   # host tensors on the device entry point
        ge.gemm_epilogue(A, B, bias)
    with pytest.raises(ValueError):
        ge.gemm_epilogue_batched(h(2, 64, 32), h(2, 32, 48), h(3, 48))      # per-item bias of the wrong batch


def test_tensor_map_cache_stats_exported(ge):
    s = ge.tensor_map_cache_stats()
    assert set(s) == {"hits", "misses"} and s["hits"] >= 0 and s["misses"] >= 0


def test_validate_round2_options(lib, ge):
    """Hadamard prologue tile, swap_ab and tile_m option checks (no device needed)."""
    S = ge.Status
    T = P * 256                                          # a fake, aligned prologue tile
    assert v(lib, opt=opts(ge, prologue=3)) == S.INVALID_VALUE                          # no tile
    assert v(lib, opt=opts(ge, prologue=3, prologue_tile=T)) == 0                       # packed ld
    assert v(lib, opt=opts(ge, prologue=3, prologue_tile=T + 2)) == S.MISALIGNED
    assert v(lib, opt=opts(ge, prologue=3, prologue_tile=T, ld_prologue_tile=60)) == S.INVALID_VALUE   # < K
    assert v(lib, opt=opts(ge, prologue=3, prologue_tile=T, ld_prologue_tile=68)) == S.MISALIGNED      # 136 B rows
    assert v(lib, opt=opts(ge, prologue=3, prologue_tile=T, ld_prologue_tile=72)) == 0
    assert v(lib, la=1, opt=opts(ge, prologue=3, prologue_tile=T, ld_prologue_tile=64)) == S.INVALID_VALUE  # < M
    assert v(lib, C=T, opt=opts(ge, prologue=3, prologue_tile=T)) == S.ALIASING        # C overlaps S
    assert v(lib, opt=opts(ge, prologue=4)) == S.INVALID_VALUE
    assert v(lib, opt=opts(ge, swap_ab=3)) == S.INVALID_VALUE
    assert v(lib, opt=opts(ge, swap_ab=2)) == 0
    assert v(lib, opt=opts(ge, tile_m=64)) == S.INVALID_VALUE
    assert v(lib, opt=opts(ge, tile_m=256, cta_group=1)) == S.INVALID_VALUE
    assert v(lib, opt=opts(ge, tile_m=128, cta_group=2, tile_n=512)) == S.INVALID_VALUE  # half-row: BN 128/256
    assert v(lib, opt=opts(ge, tile_m=128, cta_group=2, tile_n=256)) == 0


def test_plan_ex_round2_decisions(ge):
    """ge_plan_ex reports half-row pairs, multicast and swap-AB as a launch would decide them."""
    p = ge.plan(1024, 1024, 1024, tile_m=128, cta_group=2, tile_n=256)
    assert (p["tile_m"], p["tile_n"], p["cta_group"], p["num_tiles"]) == (128, 256, 2, 8 * 4)
    assert ge.plan(1024, 1024, 1024, tile_m=256)["tile_m"] in (256, 512)
    assert ge.plan(35, 8457, 2560, op="relu")["swap_ab"] == 1                        # no bias: legal
    p = ge.plan(4096, 4096, 4096, multicast=2, tile_n=256)
    assert p["multicast"] == 1 and p["tile_m"] == 512
    with pytest.raises(ge.GEError):
        ge.plan(1024, 1024, 1024, tile_m=128, cta_group=2, tile_n=64)
