"""The ordered emission's prefix arithmetic and dense-tile queue in isolation
(tools/emit_unit.cu, compiled against csrc/rk_emit.cu): synthetic per-tile counts from 1
to 2^21 tiles, with and without the queue; the total must match and the queue must come
back empty and reset after every launch."""

import shutil
import subprocess
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parents[1]


def test_emit_unit(gpu, tmp_path):
    nvcc = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    exe = tmp_path / "emit_unit"
    subprocess.run([nvcc, "-gencode", "arch=compute_100a,code=sm_100a", "-std=c++17",
                    "-I", str(ROOT / "paper_1810_01051_b200" / "csrc"),
                    str(ROOT / "tools" / "emit_unit.cu"), "-o", str(exe)], check=True,
                   timeout=300)
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0 and "bad=0" in r.stdout, r.stdout[-2000:]
