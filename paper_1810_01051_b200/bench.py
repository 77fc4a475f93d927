"""Timing harness -- drop-in for rkmatch.bench (/root/reference/pkg/src/rkmatch/bench.py).

Same names, dataclasses, validation and report formats as the reference (``AXES``,
``SweepConfig``, ``time_search``, ``speedup``, ``sweep``, ``format_csv`` / ``write_csv`` /
``write_json`` / ``format_table``, ``CorrectnessError``).  ``t_seq_ms`` and ``t_par_ms``
are the reference's wall-clock medians of ``search_sequential`` and ``search_parallel``
(host text in, Python list out -- here both run on the B200, so they include the
host->device copy of the text and the offsets' way back).  Every row is still accepted
only after both engines agree and a subsampled brute-force pass agrees
(bench.py:122-147).

The B200 adds one axis the reference cannot have: ``device_rows``, the same search
timed on the device with CUDA events (text already in HBM, ``rk_scan_async`` into a
preallocated offsets buffer).  It rides in the JSON report and the table; the CSV keeps
the reference's four columns (bench.py:37) so existing readers are unaffected.
"""

from __future__ import annotations

import csv
import io
import json
import os
import statistics
import time
from dataclasses import asdict, dataclass, field
from typing import Callable

import numpy as np

from . import _lib
from .datagen import DnaSpec, generate_tensor, make_pattern, splitmix64
from .matcher import MatchResult, search_naive, search_sequential
from .parallel import plan_launch, search_parallel
from .rkhash import hash_full

AXES = ("workers", "pattern_length", "file_size", "block_dim")

BLOCK_DIM_VALUES = (32, 64, 128, 256, 512, 1024)
PATTERN_LENGTH_VALUES = (25, 50, 100, 200, 800)
FILE_SIZE_VALUES = tuple(s * 2**20 for s in (2, 10, 20, 40))
DEFAULT_PATTERN_LENGTH = 7

CSV_COLUMNS = ("axis_value", "t_seq_ms", "t_par_ms", "speedup")


class CorrectnessError(RuntimeError):
    """A timed engine disagreed with another run or with the oracle."""


@dataclass
class TimedRun:
    median_ms: float
    times_ms: list[float]
    result: MatchResult


@dataclass
class BenchRow:
    axis_value: int
    t_seq_ms: float
    t_par_ms: float
    speedup: float


@dataclass
class DeviceRow:
    """Device-timed scan of one sweep value: median CUDA-event ms and text GB/s."""

    axis_value: int
    t_dev_ms: float
    gbps: float
    matches: int


@dataclass
class BenchReport:
    axis: str
    rows: list[BenchRow]
    environment: dict
    device_rows: list[DeviceRow] = field(default_factory=list)


@dataclass(frozen=True)
class SweepConfig:
    """Fixed parameters for the axes a sweep does not vary (bench.py:67-76)."""

    corpus: DnaSpec = DnaSpec(seed=42, length=20 * 2**20)
    pattern_length: int = DEFAULT_PATTERN_LENGTH
    pattern_source: str = "sampled"
    workers: int = 0
    block_dim: int = 256
    reps: int = 3


def time_search(impl: Callable[[bytes, bytes], MatchResult], text, pattern,
                reps: int = 3) -> TimedRun:
    """One untimed warmup, then ``reps`` timed runs that must all agree (bench.py:78-96)."""
    if reps < 1:
        raise ValueError("reps must be >= 1")
    reference = impl(text, pattern)
    times = []
    for _ in range(reps):
        t0 = time.perf_counter()
        result = impl(text, pattern)
        times.append((time.perf_counter() - t0) * 1e3)
        if result != reference:
            raise CorrectnessError("matcher output changed between repetitions")
    return TimedRun(statistics.median(times), times, reference)


def speedup(t_base: float, t_par: float) -> float:
    """Baseline-over-parallel time ratio (bench.py:99-103)."""
    if t_base <= 0 or t_par <= 0:
        raise ValueError("execution times must be positive")
    return t_base / t_par


def _verify_subsampled(text: bytes, pattern: bytes, result: MatchResult, seed: int,
                       samples: int = 4, window: int = 1 << 16) -> None:
    """Brute-force check of a timed result, outright or on seeded slices (bench.py:122-147)."""
    n, m = len(text), len(pattern)
    if n <= samples * window:
        if search_naive(text, pattern).offsets != result.offsets:
            raise CorrectnessError("timed engine disagrees with brute-force oracle")
        return
    claimed = np.asarray(result.offsets, dtype=np.int64)
    state = seed
    for _ in range(samples):
        draw, state = splitmix64(state)
        a = draw % (n - window + 1)
        b = a + window
        expected = {a + x for x in search_naive(text[a:b], pattern).offsets}
        lo, hi = np.searchsorted(claimed, [a, b - m + 1])
        got = set(claimed[lo:hi].tolist())
        if expected != got:
            raise CorrectnessError(
                f"timed engine disagrees with brute-force oracle on slice [{a}, {b})")


def time_device(text_dev, pattern: bytes, reps: int = 3) -> tuple[float, int]:
    """Median CUDA-event ms of one device-resident scan (text in HBM, offsets into a
    preallocated buffer, counters on the device) and its match count."""
    import torch

    dev = text_dev.device.index
    n, m = int(text_dev.numel()), len(pattern)
    nw = n - m + 1
    pat = np.frombuffer(pattern, dtype=np.uint8)
    hx = hash_full(pattern)
    L = _lib.lib()
    counts = torch.zeros(3, dtype=torch.int64, device=text_dev.device)
    cap = 1 << 16
    out = torch.empty(cap, dtype=torch.int64, device=text_dev.device)
    stream = torch.cuda.current_stream(dev)

    def launch():
        with _lib.acquire(dev) as ctx:
            _lib.check(L.rk_scan_async(ctx.handle, text_dev.data_ptr(), n, pat.ctypes.data, m,
                                       hx, 0, nw, out.data_ptr(), cap, 0, counts.data_ptr(),
                                       stream.cuda_stream))

    launch()  # warmup; also sizes the offsets buffer
    k = int(counts[0].item())
    if k > cap:
        cap = k
        out = torch.empty(cap, dtype=torch.int64, device=text_dev.device)
        launch()
    times = []
    for _ in range(max(reps, 1)):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        launch()
        e1.record(stream)
        e1.synchronize()
        times.append(e0.elapsed_time(e1))
    return statistics.median(times), k


def sweep(axis: str, values, config: SweepConfig = SweepConfig()) -> BenchReport:
    """Time sequential vs parallel while varying one knob per row (bench.py:150-220),
    plus the device-timed scan of the same text and pattern."""
    if axis not in AXES:
        raise ValueError(f"axis must be one of {AXES}, got {axis!r}")
    values = list(values)
    if not values:
        raise ValueError("sweep needs at least one value")
    if config.reps < 3:
        raise ValueError("reports require reps >= 3")
    base_workers = config.workers or os.cpu_count() or 1

    texts: dict[DnaSpec, tuple] = {}
    rows, device_rows = [], []
    for value in values:
        corpus = config.corpus
        m = config.pattern_length
        workers = base_workers
        block_dim = config.block_dim
        if axis == "workers":
            workers = int(value)
        elif axis == "pattern_length":
            m = int(value)
        elif axis == "block_dim":
            block_dim = int(value)
        elif axis == "file_size":
            corpus = DnaSpec(config.corpus.seed, int(value), config.corpus.alphabet)
        if corpus not in texts:
            dev = generate_tensor(corpus)
            texts[corpus] = (dev, dev.cpu().numpy().tobytes())
        text_dev, text = texts[corpus]
        pattern = make_pattern(text, corpus, m, config.pattern_source)
        cfg = plan_launch(len(text), m, block_dim)

        seq = time_search(search_sequential, text, pattern, config.reps)
        par = time_search(lambda t, p: search_parallel(t, p, cfg, workers), text, pattern,
                          config.reps)
        if seq.result != par.result:
            raise CorrectnessError(f"sequential and parallel engines disagree at {axis}={value}")
        _verify_subsampled(text, pattern, seq.result, corpus.seed)
        rows.append(BenchRow(value, seq.median_ms, par.median_ms,
                             speedup(seq.median_ms, par.median_ms)))
        if len(text) >= m:
            t_dev, k = time_device(text_dev, pattern, config.reps)
            if k != len(seq.result.offsets):
                raise CorrectnessError(f"device-timed scan disagrees at {axis}={value}")
            device_rows.append(DeviceRow(value, t_dev, len(text) / t_dev / 1e6, k))

    environment = {
        "cpu_count": os.cpu_count(),
        "workers": base_workers,
        "block_dim": config.block_dim,
        "pattern_length": config.pattern_length,
        "pattern_source": config.pattern_source,
        "reps": config.reps,
        "warmup_runs": 1,
        "corpus": {
            "seed": config.corpus.seed,
            "length": config.corpus.length,
            "alphabet": config.corpus.alphabet.decode("ascii", "replace"),
        },
        "engine": "b200",
        "device": _device_name(),
    }
    return BenchReport(axis, rows, environment, device_rows)


def _device_name() -> str:
    import torch

    return torch.cuda.get_device_name(_lib.default_device())


def format_csv(report: BenchReport) -> str:
    """axis_value,t_seq_ms,t_par_ms,speedup rows (bench.py:223-230)."""
    buf = io.StringIO()
    writer = csv.writer(buf, lineterminator="\n")
    writer.writerow(CSV_COLUMNS)
    for row in report.rows:
        writer.writerow([row.axis_value, row.t_seq_ms, row.t_par_ms, row.speedup])
    return buf.getvalue()


def write_csv(report: BenchReport, path) -> None:
    with open(path, "w", newline="") as fh:
        fh.write(format_csv(report))


def report_payload(report: BenchReport) -> dict:
    """The reference JSON report (bench.py:238-248) plus ``device_rows``."""
    return {
        "axis": report.axis,
        "rows": [asdict(row) for row in report.rows],
        "environment": report.environment,
        "device_rows": [asdict(row) for row in report.device_rows],
    }


def write_json(report: BenchReport, path) -> None:
    with open(path, "w") as fh:
        json.dump(report_payload(report), fh, indent=2)
        fh.write("\n")


def format_table(report: BenchReport) -> str:
    """Fixed-width table (bench.py:251-260), with the device-timed columns appended."""
    dev = {r.axis_value: r for r in report.device_rows}
    header = (f"{report.axis:>14}  {'t_seq_ms':>12}  {'t_par_ms':>12}  {'speedup':>9}"
              f"  {'t_dev_ms':>10}  {'dev_GB/s':>9}")
    lines = [header, "-" * len(header)]
    for row in report.rows:
        d = dev.get(row.axis_value)
        tail = f"  {d.t_dev_ms:>10.4f}  {d.gbps:>9.1f}" if d else f"  {'-':>10}  {'-':>9}"
        lines.append(f"{row.axis_value:>14}  {row.t_seq_ms:>12.3f}  {row.t_par_ms:>12.3f}"
                     f"  {row.speedup:>9.4f}" + tail)
    return "\n".join(lines)
