"""Build the sm_100a shared library libgemm_epilogue.so in-tree with nvcc (no JIT cache).

Each instantiation unit compiles in parallel; the C-ABI runtime links the CUDA runtime
statically so the library does not depend on which libcudart the host process loaded."""
from __future__ import annotations

import concurrent.futures as cf
import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(PKG, "csrc")
ROOT = os.path.dirname(PKG)
LIB = os.path.join(PKG, "libgemm_epilogue.so")
BUILD = os.path.join(PKG, "build")
# Diagnostics variant (GE_DEBUG_STATS=1 loads it): per-role barrier-wait counters compiled in.
LIB_DBG = os.path.join(PKG, "libgemm_epilogue_dbg.so")
BUILD_DBG = os.path.join(PKG, "build_dbg")

NVCC = os.environ.get("NVCC", shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-Xcompiler", "-Wall",
         "--expt-relaxed-constexpr", "-I", os.path.join(ROOT, "include")]


def sources():
    return sorted(os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith(".cu"))


def _deps():
    return [os.path.join(CSRC, f) for f in os.listdir(CSRC)] + [os.path.join(ROOT, "include", "gemm_epilogue.h")]


def up_to_date(lib: str = LIB) -> bool:
    if not os.path.exists(lib):
        return False
    t = os.path.getmtime(lib)
    return all(os.path.getmtime(d) <= t for d in _deps())


def build(force: bool = False, verbose: bool = False, extra=None, debug_stats: bool = False,
          variant: str = "") -> str:
    """variant: dev A/B builds (libgemm_epilogue_<variant>.so, objects under build_<variant>/)."""
    lib, bdir = (LIB_DBG, BUILD_DBG) if debug_stats else (LIB, BUILD)
    if variant:
        lib = os.path.join(PKG, f"libgemm_epilogue_{variant}.so")
        bdir = os.path.join(PKG, f"build_{variant}")
    if not force and up_to_date(lib):
        return lib
    os.makedirs(bdir, exist_ok=True)
    extra = list(extra or []) + (["-DGE_DBG=1"] if debug_stats else [])

    def comp(src):
        obj = os.path.join(bdir, os.path.basename(src) + ".o")
        cmd = [NVCC, *ARCH, *FLAGS, *extra, "-c", src, "-o", obj]
        if verbose:
            print(" ".join(cmd), flush=True)
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed on {src}:\n{r.stdout}\n{r.stderr}")
        if verbose and (r.stdout or r.stderr):
            print(r.stdout, r.stderr, flush=True)
        return obj

    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 4)) as ex:
        objs = list(ex.map(comp, sources()))
    tmp = lib + f".tmp{os.getpid()}"
    cmd = [NVCC, *ARCH, "-shared", "-cudart", "static", "-o", tmp, *objs, "-lcuda" if False else "-ldl"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    # dev: --variant NAME -DFOO=1 ... builds libgemm_epilogue_NAME.so with extra defines
    var = sys.argv[sys.argv.index("--variant") + 1] if "--variant" in sys.argv else ""
    defs = [a for a in sys.argv if a.startswith("-D")]
    print(build(force="--force" in sys.argv or bool(var), verbose=True,
                extra=(["-Xptxas", "-v"] if "--ptxas-v" in sys.argv else []) + defs,
                debug_stats="--debug-stats" in sys.argv, variant=var))
