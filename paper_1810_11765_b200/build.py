"""Build libdsr.so in-tree with nvcc for sm_100a (no JIT cache, no torch types).

    python -m paper_1810_11765_b200.build [--force]
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys
import time
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
OUT = PKG / "libdsr.so"
BUILD = PKG / "_build"
SOURCES = ["capi.cu", "app_microbench.cu", "app_gol.cu", "app_wator.cu", "app_wator_static.cu", "app_nbody.cu"]
HEADERS = ["dsr_device.cuh", "dsr_doall.cuh", "dsr_host.h"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-Wall",
         "--expt-relaxed-constexpr", "-Xptxas", "-warn-spills"]
# N-body: r^2 >= eps^2 is never denormal, so flush-to-zero lets rsqrtf be a bare
# MUFU.RSQ (no per-pair denormal fix-up in the all-pairs loops)
PER_FILE = {"app_nbody.cu": ["-ftz=true"]}


def _git_rev() -> str:
    try:
        return subprocess.run(["git", "-C", str(ROOT), "rev-parse", "--short", "HEAD"], capture_output=True,
                              text=True, timeout=10).stdout.strip() or "nogit"
    except Exception:
        return "nogit"


def src_hash() -> str:
    """sha1 (12 hex) of the library's sources and header: identifies a build
    independently of git (the GPU box gets the tree without .git); profiles
    record it so bench.py only reuses ncu counts of the same code."""
    import hashlib
    h = hashlib.sha1()
    for f in [CSRC / s for s in SOURCES + HEADERS] + [ROOT / "include" / "dsr.h"]:
        h.update(f.read_bytes())
    return h.hexdigest()[:12]


def _stale() -> bool:
    if not OUT.exists():
        return True
    t = OUT.stat().st_mtime
    deps = [CSRC / s for s in SOURCES + HEADERS] + [ROOT / "include" / "dsr.h", Path(__file__)]
    return any(d.stat().st_mtime > t for d in deps)


def build(force: bool = False, verbose: bool = False, profile: bool = False, variant: str = "",
          defines=()) -> Path:
    """profile=True: a second library, _build/libdsr_prof.so, compiled with
    -DDSR_PROFILE (request-level allocator counters; load it with
    DSR_LIBPATH=... for scripts/prof_mb.py).  The product library has none.
    variant/defines: an experiment build _build/libdsr_<variant>.so with extra
    -D definitions (tuning sweeps through DSR_LIBPATH)."""
    tag = "prof" if profile else variant
    out = BUILD / f"libdsr_{tag}.so" if tag else OUT
    if not force and not tag and not _stale():
        return OUT
    BUILD.mkdir(exist_ok=True)
    info = f'-DDSR_BUILD_INFO="sm_100a src:{src_hash()} {_git_rev()} {time.strftime("%Y-%m-%d")}"'
    extra = (["-DDSR_PROFILE"] if profile else []) + [f"-D{d}" for d in defines]

    def compile_one(src: str) -> Path:
        obj = BUILD / (Path(src).stem + (f"_{tag}" if tag else "") + ".o")
        cmd = [NVCC, *ARCH, *FLAGS, *extra, *PER_FILE.get(src, []), info, "-I", str(ROOT / "include"), "-c",
               str(CSRC / src), "-o", str(obj)]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
        if verbose and (r.stdout or r.stderr):
            print(r.stdout, r.stderr, file=sys.stderr)
        return obj

    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        objs = list(ex.map(compile_one, SOURCES))
    tmp = out.with_suffix(".so.tmp")
    cmd = [NVCC, *ARCH, "-shared", "-o", str(tmp), *map(str, objs), "-lcuda"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    os.replace(tmp, out)
    return out


if __name__ == "__main__":
    t0 = time.time()
    p = build(force="--force" in sys.argv, verbose=True, profile="--profile" in sys.argv)
    print(f"built {p} in {time.time() - t0:.1f}s")
