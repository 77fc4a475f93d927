"""Build librkb200.so in-tree with nvcc for sm_100a (no JIT cache, no torch arch list).

    python -m paper_1810_01051_b200._build [--force]

Each .cu is compiled in parallel to an object under build/, then linked with the static
CUDA runtime into paper_1810_01051_b200/librkb200.so.  Rebuilds only when a source or
header is newer than the library.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
# RK_DEFINES / RK_LIB_OUT: build a variant library (extra -D flags, another output path)
# for A/B timing with tools/ (the package itself always loads librkb200.so)
BUILD = ROOT / "build" / ("rkb200" + os.environ.get("RK_LIB_TAG", ""))
LIB = Path(os.environ["RK_LIB_OUT"]).resolve() if os.environ.get("RK_LIB_OUT") else PKG / "librkb200.so"
DEFINES = os.environ.get("RK_DEFINES", "").split()
SOURCES = ["rk_scan.cu", *[f"rk_scan_g{g}.cu" for g in range(4)], "rk_multi.cu",
           "rk_multi_g0.cu", "rk_pairs.cu", "rk_emit.cu", "rk_aux.cu", "rk_capi.cu", "rk_comm.cu"]
HEADERS = ["rk_device.cuh", "rk_internal.h", "rk_scan_impl.cuh", "rk_short_impl.cuh", "rk_multi_impl.cuh", "rk_ctx.h"]

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVFLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O3", "--use_fast_math",
           "-Xptxas", "-warn-spills"]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found; the B200 build needs CUDA 12.9's nvcc")


def _stale() -> bool:
    if not LIB.exists():
        return True
    t = LIB.stat().st_mtime
    deps = [CSRC / s for s in SOURCES + HEADERS] + [ROOT / "include" / "rkb200.h"]
    return any(d.stat().st_mtime > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> Path:
    if not force and not _stale():
        return LIB
    BUILD.mkdir(parents=True, exist_ok=True)
    cc = nvcc()
    inc = ["-I", str(ROOT / "include"), "-I", str(CSRC)]

    def compile_one(src: str) -> Path:
        obj = BUILD / (Path(src).stem + ".o")
        cmd = [cc, *ARCH, *NVFLAGS, *DEFINES, *inc, "-c", str(CSRC / src), "-o", str(obj)]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
        if verbose and (r.stdout or r.stderr):
            print(r.stdout, r.stderr, file=sys.stderr)
        return obj

    with ThreadPoolExecutor(max_workers=min(len(SOURCES), os.cpu_count() or 4)) as ex:
        objs = list(ex.map(compile_one, SOURCES))
    tmp = LIB.with_suffix(".so.tmp")
    cmd = [cc, *ARCH, "-shared", "-cudart", "static", "-o", str(tmp), *map(str, objs),
           "-lpthread", "-ldl", "-lrt"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
