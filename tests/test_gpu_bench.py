"""The benchmark driver itself (bench.py): the default single-GPU line carries the contract's
keys, and the multi-rank path runs under torchrun -- here as its one-GPU plumbing test
(two ranks on cuda:0 exchanging through gloo on the host; no rank waits on another's
kernels)."""

import json
import os
import socket
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parent.parent
SMALL = ["--bytes-per-gpu", str(64 << 20), "--steps", "3", "--warmup", "3", "--no-cpu",
         "--e2e-steps", "1", "--sustained-steps", "3", "--pass-gap", "0"]


def _run(cmd, timeout=600):
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=timeout)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [x for x in r.stdout.splitlines() if x.startswith("{")]
    return [json.loads(x) for x in lines]


def test_bench_single_gpu_line(gpu):
    (line,) = _run([sys.executable, "bench.py", *SMALL])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "vs_baseline", "dtype", "config", "roofline",
              "e2e", "clocks", "gpu_launches", "sustained"):
        assert k in line, k
    assert line["n_gpus"] == 1 and line["value"] > 0 and line["gpu_launches"] > 0
    assert line["e2e"]["api"].startswith("rk_scan_host_batch")
    assert line["e2e"]["h2d_bytes_per_step"] >= 64 << 20
    assert set(line["per_m_gbs"]) == {"4", "8", "16", "32", "64", "128", "256", "512", "1024"}


def test_bench_two_rank_plumbing(gpu):
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    lines = _run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                  "--nproc-per-node", "2", "--master-addr", "127.0.0.1", "--master-port",
                  str(port), "bench.py", "--gpus", "2", "--same-device", "--dist-backend",
                  "gloo", *SMALL])
    assert len(lines) == 1  # rank 0 alone prints
    line = lines[0]
    assert line["n_gpus"] == 2 and line["scaling"] == "weak" and line["value"] > 0


def test_bench_exchange_path_one_rank(gpu):
    """The N > 1 step's exchange (rk_scan_sharded_batch_async through the C-ABI NCCL
    communicator, no host round trip per step) run at one rank: the line reports it, the
    counts it gathered match the plain path's, and a slab too small for a list falls back
    to the synchronous batch."""
    (plain,) = _run([sys.executable, "bench.py", *SMALL])
    (line,) = _run([sys.executable, "bench.py", "--force-comm", *SMALL])
    assert line["exchange"]["api"].startswith("rk_scan_sharded_batch_async")
    assert line["matches_per_m"] == plain["matches_per_m"] and line["value"] > 0
    (small,) = _run([sys.executable, "bench.py", "--force-comm", "--slab", "1", *SMALL])
    over = max(plain["matches_per_m"].values()) > 1
    assert small["exchange"]["api"].startswith(
        "rk_scan_sharded_batch (" if over else "rk_scan_sharded_batch_async")
    assert small["matches_per_m"] == plain["matches_per_m"]
