#!/usr/bin/env python
"""Benchmark: text scanned GB/s on B200 (BASELINE.json `metric`), one JSON line.

Workload (BASELINE.json configs[1], "C2"): 1 GiB of synthetic printable-ASCII text per
GPU (the reference generator, seed 42, produced on the device), single-pattern scans for
the pattern-length sweep m = 4, 8, 16, 32, 64, 128, 256, 512, 1024 (patterns sampled
from the corpus as rkmatch.bench._make_pattern does).  One step = the whole sweep, i.e.
9 full scans of the text; value = text bytes scanned by all ranks / device time.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

N > 1 runs under torchrun, one rank per GPU: weak scaling, each rank owns 1 GiB of the
global N GiB corpus plus an (m-1)-byte halo, scans it, and the global ordered position
lists are returned to every rank by the C ABI's rk_scan_sharded_batch_async (one NCCL
group per step, no host round trip).
`--workload C4` runs BASELINE configs[3] instead: 16 GiB DNA, m = 32, strong scaling.  `--impl reference` times the reference
algorithm (the C restatement in oracle/ of rkmatch._scan_range + search_parallel's range
partition) on the host cores on a bounded sample of the same workload.
"""

from __future__ import annotations

import argparse
import ctypes
import json
import os
import statistics
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "text scanned GB/s (device-timed) at 1/2/4/8 B200 vs HBM roofline; host-CPU ref GB/s"
SWEEP = (4, 8, 16, 32, 64, 128, 256, 512, 1024)
ASCII = bytes(range(32, 127))
SEED = 42
GiB = 1 << 30


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--bytes-per-gpu", type=int, default=GiB)
    ap.add_argument("--sweep", type=str, default=",".join(map(str, SWEEP)))
    ap.add_argument("--e2e-steps", type=int, default=None)
    ap.add_argument("--workload", choices=("C2", "C4"), default="C2",
                    help="C2 (default, BASELINE configs[1], weak scaling) or C4 (configs[3]: "
                         "16 GiB DNA, strong scaling)")
    ap.add_argument("--c4-bytes", type=int, default=16 * GiB)
    ap.add_argument("--sustained-steps", type=int, default=200)
    ap.add_argument("--force-comm", action="store_true",
                    help="run the N > 1 exchange path (C-ABI communicator) even at one rank (tests)")
    ap.add_argument("--slab", type=int, default=4096,
                    help="N > 1: offsets per pattern and rank exchanged without a host round trip")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--ref-seconds", type=float, default=150.0,
                    help="--impl reference: host-CPU budget of the whole run")
    # test plumbing only: exercise the multi-rank path on a one-GPU box (all ranks on
    # cuda:0, gloo instead of NCCL so no collective kernels wait on each other there)
    ap.add_argument("--dist-backend", default="nccl", choices=("nccl", "gloo"))
    ap.add_argument("--same-device", action="store_true")
    ap.add_argument("--lib", default=None, help=argparse.SUPPRESS)  # A/B of a variant build
    ap.add_argument("--pass-gap", type=float, default=1.0, help=argparse.SUPPRESS)
    return ap.parse_args()


# ------------------------------------------------------------------------- helpers
def load_peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


class ClockSampler:
    """SM clock + throttle reasons via NVML, sampled during the timed region."""

    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
        0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
        0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
        0x100: "display_clock_setting",
    }

    def __init__(self, device: int):
        self.samples: list[int] = []
        self.reasons: int = 0
        self.max_mhz = None
        self._stop = threading.Event()
        self._t = None
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                self.reasons |= int(self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h))
            except Exception:
                pass
            time.sleep(0.0005)

    def __enter__(self):
        if self.nv is not None:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
            t0 = time.time()
            while not self.samples and time.time() - t0 < 1.0:  # sampler is running
                time.sleep(0.0002)
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unavailable"]}
        names = [v for k, v in self.REASONS.items() if self.reasons & k and k != 0x1]
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": names, "samples": len(self.samples)}


def sampled_offset(n_total: int, m: int) -> int:
    """rkmatch.bench._make_pattern 'sampled' position (bench.py:112-114)."""
    from paper_1810_01051_b200.datagen import splitmix64

    draw, _ = splitmix64(SEED ^ 0xA5A5A5A5A5A5A5A5)
    return draw % (n_total - m + 1)


# ------------------------------------------------------------------------- CPU arm
def cpu_rates(text: np.ndarray, patterns: dict, seconds: float, threads: int):
    """Time the reference algorithm (oracle C port of _scan_range + search_parallel's
    range partition) on prefixes sized for ~seconds/len(patterns) each."""
    import oracle

    per = seconds / len(patterns)
    sec_per_byte = 0.0  # equal bytes per m, as in the GPU sweep: harmonic combination
    sample = {}
    for m, pat in patterns.items():
        p = np.frombuffer(pat, dtype=np.uint8)
        size = 1 << 20
        while True:
            t0 = time.perf_counter()
            oracle.c_scan(text[:size], p, workers=threads)
            dt = time.perf_counter() - t0
            if dt >= per * 0.5 or size >= text.size:
                break
            size = int(min(text.size, size * max(2.0, per / max(dt, 1e-4))))
        sec_per_byte += dt / size
        sample[m] = size
    return len(patterns) / sec_per_byte / 1e9, sample


def cpu_fixed(text, patterns, sizes, threads):
    import oracle

    sec_per_byte = 0.0
    t_all = 0.0
    for m, pat in patterns.items():
        t0 = time.perf_counter()
        oracle.c_scan(text[: sizes[m]], np.frombuffer(pat, dtype=np.uint8), workers=threads)
        dt = time.perf_counter() - t0
        t_all += dt
        sec_per_byte += dt / sizes[m]
    return sec_per_byte, t_all


def workload_config(per: int, sweep, world: int) -> dict:
    """The workload both arms report (BASELINE.json configs[1])."""
    return {"workload": "C2: single-pattern length sweep over 1 GiB printable-ASCII "
                        "text per GPU (BASELINE.json configs[1])",
            "bytes_per_gpu": per, "sweep": sweep, "pattern_source": "sampled",
            "corpus": "DnaSpec(42, N GiB, bytes(32..126))",
            "l2": "inputs larger than L2 (1 GiB per GPU vs 126 MB)",
            "parallelism": f"shard{world} (contiguous, (m-1)-byte halo)"}


def run_reference(args):
    """--impl reference: the reference algorithm on the host cores, same metric."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import oracle

    sweep = [int(x) for x in args.sweep.split(",")]
    threads = oracle.cpu_threads()
    n = 256 << 20
    text = np.frombuffer(oracle.generate(SEED, n, ASCII), dtype=np.uint8)
    pats = {m: text[sampled_offset(n, m): sampled_offset(n, m) + m].tobytes() for m in sweep}
    # per-step sample sizes so that the run (warmup + steps) stays within minutes
    budget = max(min(2.0, args.ref_seconds), args.ref_seconds / max(1, args.steps + args.warmup))
    _, sizes = cpu_rates(text, pats, budget, threads)
    for _ in range(args.warmup):
        cpu_fixed(text, pats, sizes, threads)
    times = []
    spb = 0.0
    for _ in range(args.steps):
        sb, dt = cpu_fixed(text, pats, sizes, threads)
        times.append(dt)
        spb += sb
    total = sum(times)
    # equal bytes per pattern length (the GPU sweep's weighting): harmonic combination
    gbs = len(sweep) * args.steps / spb / 1e9
    line = {
        "impl": "reference", "metric": METRIC, "value": gbs, "unit": "GB/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": total / args.steps * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "u8", "data": "synthetic",
        "config": workload_config(args.bytes_per_gpu, sweep, args.gpus),
        "cpu_baseline": {"value": gbs, "unit": "GB/s", "cores": threads, "kind": "port",
                         "sample": f"per step, prefixes {sizes} (bytes per m) of the C2 corpus; "
                                   f"oracle C port of _scan_range + search_parallel ranges"},
        "e2e": {"value": gbs, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------------- GPU arm
def load_traffic():
    """Per-m DRAM bytes per launch of rk_scan_kernel<M> (dram__bytes_read.sum +
    dram__bytes_write.sum), from the ncu pass of this command summarised by
    profiles/traffic_from_ncu.py."""
    p = ROOT / "profiles" / "r02_traffic.json"
    if not p.exists():
        return None
    try:
        return json.loads(p.read_text())
    except Exception:
        return None


def setup_dist(args):
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    dev = 0 if args.same_device else local
    torch.cuda.set_device(dev)
    if world > 1:
        # each rank logs its NCCL communicator (torch's and librkb200's) to stderr
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
        os.environ.setdefault("RKB200_COMM_LOG", "1")
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device(f"cuda:{dev}"))
        else:
            dist.init_process_group("gloo")
    return world, rank, dev


def timed_steps(step, steps, stream, dev, world):
    """K steps back to back bracketed by a barrier + synchronize, device-timed with CUDA
    events on the launching stream, max over ranks; NVML clocks sampled meanwhile."""
    import torch
    import torch.distributed as dist

    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(dev) as clk:
        start.record(stream)
        for _ in range(steps):
            step(None)
        end.record(stream)
        # poll (sleeping, GIL released) instead of blocking, so the clock sampler thread
        # keeps sampling while the device drains the queued steps
        while not end.query():
            time.sleep(0.0002)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    t = torch.tensor([start.elapsed_time(end)], dtype=torch.float64, device=f"cuda:{dev}")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item()), clk.summary()


def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_1810_01051_b200 as rk
    from paper_1810_01051_b200 import _lib, _scan, sharded

    if args.lib:
        _lib.LIB_PATH = Path(args.lib).resolve()
    world, rank, dev = setup_dist(args)
    if args.workload == "C4":
        return run_c4(args, world, rank, dev)
    sweep = [int(x) for x in args.sweep.split(",")]
    per = args.bytes_per_gpu
    n_total = per * world
    mmax = max(sweep)
    spec = rk.DnaSpec(SEED, n_total, ASCII)

    # this rank's bytes: [rank*per, rank*per + per + mmax - 1) ∩ [0, n_total)
    byte_lo = rank * per
    byte_hi = min(n_total, byte_lo + per + mmax - 1)
    text = rk.generate_tensor(spec, device=f"cuda:{dev}", skip=byte_lo, count=byte_hi - byte_lo)
    pats, plans = {}, {}
    for m in sweep:
        x = sampled_offset(n_total, m)
        pats[m] = rk.generate_tensor(spec, device=f"cuda:{dev}", skip=x, count=m).cpu().numpy().tobytes()
        a, b, blo, bhi = sharded.weak_shard(rank, per, n_total, m)
        plans[m] = (a - byte_lo, b - byte_lo, rk.hash_full(pats[m]))
    L = _lib.lib()
    ctx = _lib.context(dev)
    # N > 1: the exchange through the C ABI (NCCL); --dist-backend gloo (the plumbing test of
    # this multi-rank path on one GPU: ranks never wait on each other's kernels) exchanges
    # through torch.distributed on the host instead
    comm = (sharded.Communicator(device=dev)
            if (world > 1 and args.dist_backend == "nccl") or args.force_comm else None)
    gloo = world > 1 and comm is None
    stream = torch.cuda.current_stream(dev)
    sptr = stream.cuda_stream
    cap = 1 << 22
    out_all = torch.empty((len(sweep), cap), dtype=torch.int64, device=f"cuda:{dev}")
    outs = {m: out_all[i] for i, m in enumerate(sweep)}
    counts = torch.zeros((len(sweep), 3), dtype=torch.int64, device=f"cuda:{dev}")
    glob = {}
    pat_bufs = {m: np.frombuffer(pats[m], dtype=np.uint8) for m in sweep}
    n_local = int(text.numel())
    acounts = torch.zeros((len(sweep), 4), dtype=torch.int64, device=f"cuda:{dev}")
    batch_async = [comm is not None]  # N > 1 over NCCL: the asynchronous batch

    def step(ev_pairs=None):
        for i, m in enumerate(sweep):
            a, b, hx = plans[m]
            if ev_pairs is not None:
                ev_pairs[i][0].record(stream)
            if comm is not None:
                if ev_pairs is None:
                    continue  # the whole sweep's exchange in one call, below
                # (the per-length pass times each length's own collective)
                glob[m] = comm.scan(text, pats[m], a + byte_lo, b + byte_lo, byte_lo,
                                    cap=cap, out=outs[m], stream=sptr)
            elif gloo:
                def scan_fn(t, p, lo, hi, hx=hx):
                    o, k, co, hh = _scan.scan_counts(t, p, hx, lo, hi)
                    return o.cpu(), k, co, hh
                allo, tot = sharded.search_sharded(text, pats[m], a + byte_lo, b + byte_lo, byte_lo,
                                                   scan_fn=scan_fn)
                glob[m] = (allo, tot[0], tot[2], tot[1])
            elif comm is None:
                _lib.check(L.rk_scan_async(ctx.handle, text.data_ptr(), n_local,
                                           pat_bufs[m].ctypes.data, m, hx, a, b,
                                           outs[m].data_ptr(), cap, byte_lo,
                                           counts[i].data_ptr(), sptr))
            if ev_pairs is not None:
                ev_pairs[i][1].record(stream)
        if comm is not None and ev_pairs is None:
            if batch_async[0]:
                # the C ABI's asynchronous batched sharded scan: the nine local scans back to
                # back, each into a fixed slab, then ONE NCCL group all-gathering every rank's
                # counters and slabs, and a device kernel ordering every rank's positions
                # into every rank's outputs -- no host round trip inside the step
                comm.scan_batch_async(text, [pats[m] for m in sweep],
                                      [(plans[m][0] + byte_lo, plans[m][1] + byte_lo)
                                       for m in sweep],
                                      byte_lo, [outs[m] for m in sweep], acounts,
                                      slab=args.slab, stream=sptr)
            else:
                # (a rank found more than a slab: the synchronous batch, which sizes the
                # exchange from the gathered counts)
                res = comm.scan_batch(text, [pats[m] for m in sweep],
                                      [(plans[m][0] + byte_lo, plans[m][1] + byte_lo)
                                       for m in sweep],
                                      byte_lo, [outs[m] for m in sweep], stream=sptr)
                for m, r in zip(sweep, res):
                    glob[m] = r
        return counts

    for _ in range(max(args.warmup, 3)):
        step()
    torch.cuda.synchronize()
    if comm is not None and batch_async[0]:
        ac = acounts.cpu().numpy()
        if ac[:, 3].any():
            batch_async[0] = False  # some list is over a slab: the synchronous batch
            for _ in range(max(args.warmup, 3)):
                step()
            torch.cuda.synchronize()
        else:
            for i, m in enumerate(sweep):
                glob[m] = (outs[m][: int(ac[i, 0])], int(ac[i, 0]), int(ac[i, 2]), int(ac[i, 1]))
    # correctness gate: counts add up; at N > 1 every rank holds the same global ascending
    # list, and its total is the sum over ranks
    if comm is None and not gloo:
        host_counts = counts.cpu().numpy()
    else:
        host_counts = np.array([[glob[m][1], glob[m][3], glob[m][2]] for m in sweep], dtype=np.int64)
        for m in sweep:
            g = glob[m][0]
            assert g.numel() == glob[m][1] and bool((g[1:] > g[:-1]).all())
    assert (host_counts[:, 1] == host_counts[:, 0] + host_counts[:, 2]).all()

    # Headline: K steps back to back with nothing between the launches (an event recorded
    # between two kernels costs the programmatic-dependent-launch overlap, ~4%).  Then,
    # after an idle gap (right after ~30 ms of full-bandwidth streaming the next pass runs
    # ~4% slower; after ~1 s idle it does not), the same K steps again with CUDA events
    # around every scan + emit, for the per-length numbers and the kernel's per-launch
    # duration (roofline).  Last, a sustained pass of many steps (power-capped clocks).
    ev = [[(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in sweep] for _ in range(args.steps)]
    launches0 = ctx.launches + (comm.ctx.launches if comm else 0)
    elapsed_ms, clk = timed_steps(step, args.steps, stream, dev, world)
    launches = ctx.launches + (comm.ctx.launches if comm else 0) - launches0
    time.sleep(args.pass_gap)
    # per-length pass: the same steps with events around every scan + emit
    with ClockSampler(dev) as clk_b:
        for s in range(args.steps):
            step(ev[s])
        while not ev[-1][-1][1].query():
            time.sleep(0.0002)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    per_m_ms = {m: sum(ev[s][i][0].elapsed_time(ev[s][i][1]) for s in range(args.steps)) / args.steps
                for i, m in enumerate(sweep)}
    windows_all = sum(max(n_total - m + 1, 0) for m in sweep)
    value = windows_all / (elapsed_ms / args.steps / 1e3) / 1e9  # text (window) bytes/s
    sustained = None
    if args.sustained_steps > 0:
        time.sleep(args.pass_gap)
        sus_ms, clk_s = timed_steps(step, args.sustained_steps, stream, dev, world)
        sustained = {"value": windows_all / (sus_ms / args.sustained_steps / 1e3) / 1e9,
                     "unit": "GB/s", "steps": args.sustained_steps,
                     "ms_per_step": sus_ms / args.sustained_steps, "clocks": clk_s,
                     "note": "the headline's steps back to back for ~0.3 s: the board's power "
                             "limit lowers the SM clock under sustained full-bandwidth streaming"}

    # roofline of the scan kernel: algorithmic bytes = n + 8*matches per launch (local)
    peak, peak_kind = load_peaks()
    local_counts = counts.cpu().numpy() if comm is None and not gloo else None
    alg = [(plans[m][1] - plans[m][0] + m - 1) +
           8 * int((local_counts if local_counts is not None else host_counts)[i, 0])
           for i, m in enumerate(sweep)]
    achieved = sum(alg) / (sum(per_m_ms.values()) / 1e3) / 1e9
    tr = load_traffic()
    traffic = traffic_per_m = None
    if tr and all(str(m) in tr.get("per_m", {}) for m in sweep):
        traffic_per_m = {str(m): tr["per_m"][str(m)] for m in sweep}
        traffic = sum(traffic_per_m.values()) / len(sweep)  # per launch, sweep mean

    # ---------------------------------------------------------------- e2e (host API)
    # search_each's C entry point, rk_scan_host_batch: this rank's text from pinned host
    # memory and the sweep's patterns in, every pattern's counters and ordered offsets
    # back in host memory; the text crosses PCIe once per step and each pattern's windows
    # are scanned as their bytes land (a step's inputs copied every step, inside the
    # timed region).  e2e_per_call: rk_scan_host per pattern (search_sequential on a host
    # text: the text crosses PCIe for every pattern).
    e2e_steps = args.e2e_steps if args.e2e_steps is not None else min(args.steps, 3)
    e2e = e2e_call = None
    if e2e_steps > 0:
        host = text.cpu().pin_memory()
        h_out = torch.empty(1 << 20, dtype=torch.int64).pin_memory()
        flat = np.frombuffer(b"".join(pats[m] for m in sweep), dtype=np.uint8)
        lens = np.array(sweep, dtype=np.uint32)
        hashes = np.array([plans[m][2] for m in sweep], dtype=np.uint64)
        b_mt, b_co, b_hh = (np.zeros(len(sweep), dtype=np.uint64) for _ in range(3))
        mt, co, hh = _lib.u64ref(), _lib.u64ref(), _lib.u64ref()
        h2d = d2h = 0
        # (the batch call scans every window of the text it is given: at N > 1 a rank's
        # text ends with its (mmax - 1)-byte halo, so shorter patterns also see a few of the
        # next rank's windows there -- an end-to-end rank-local number, not an exchange)

        def e2e_step():
            nonlocal h2d, d2h
            _lib.check(L.rk_scan_host_batch(ctx.handle, host.data_ptr(), n_local,
                                            flat.ctypes.data, lens.ctypes.data,
                                            hashes.ctypes.data, len(sweep), h_out.data_ptr(),
                                            h_out.numel(), b_mt.ctypes.data, b_co.ctypes.data,
                                            b_hh.ctypes.data))
            h2d += n_local + int(flat.size)
            d2h += 8 * min(int(b_mt.sum()), h_out.numel()) + 32 * len(sweep)
            return [int(v) for v in b_mt]

        def e2e_call_step():
            nonlocal h2d, d2h
            got = []
            for m in sweep:
                a, b, hx = plans[m]
                _lib.check(L.rk_scan_host(ctx.handle, host.data_ptr(), n_local, pat_bufs[m].ctypes.data,
                                          m, hx, a, b, h_out.data_ptr(), h_out.numel(),
                                          ctypes.byref(mt), ctypes.byref(co), ctypes.byref(hh)))
                h2d += (b - a) + m - 1
                d2h += 8 * min(int(mt.value), h_out.numel()) + 24
                got.append(int(mt.value))
            return got

        def timed_e2e(fn, steps, api, check):
            nonlocal h2d, d2h
            got = fn()
            if check is not None:
                assert got == check, (got, check)
            h2d = d2h = 0
            torch.cuda.synchronize()
            if world > 1:
                dist.barrier()
            t0 = time.perf_counter()
            for _ in range(steps):
                fn()
            torch.cuda.synchronize()
            t_e = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device=f"cuda:{dev}")
            if world > 1:
                dist.all_reduce(t_e, op=dist.ReduceOp.MAX)
            return {"value": windows_all / (float(t_e.item()) / steps) / 1e9, "unit": "GB/s",
                    "h2d_bytes_per_step": h2d // steps, "d2h_bytes_per_step": d2h // steps,
                    "steps": steps, "api": api}

        local_k = [int(v) for v in (local_counts[:, 0] if local_counts is not None else [0] * len(sweep))]
        e2e = timed_e2e(e2e_step, e2e_steps,
                        "rk_scan_host_batch (C ABI; Python: paper_1810_01051_b200.search_each) -- "
                        "pinned host text + the 9 patterns in, per-pattern counters and ordered "
                        "offsets out in host memory; the text crosses PCIe once per step in 64 "
                        "MiB chunks, every pattern scanning each chunk as it lands",
                        local_k if local_counts is not None else None)
        e2e_call = timed_e2e(e2e_call_step, 1,
                             "rk_scan_host per pattern (search_sequential on a host text: the "
                             "text crosses PCIe for every pattern, chunked DMA overlapped with "
                             "the scan)", local_k if local_counts is not None else None)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        import oracle

        threads = oracle.cpu_threads()
        host_text = text[: 256 << 20].cpu().numpy()
        rate, sample = cpu_rates(host_text, {m: pats[m] for m in sweep}, args.cpu_seconds, threads)
        cpu = {"value": rate, "unit": "GB/s", "cores": threads, "kind": "port",
               "sample": f"prefixes of the C2 corpus per m: {sample} bytes (oracle C port of "
                         f"_scan_range + search_parallel ranges, {threads} threads)"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": elapsed_ms / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "u8",
            "data": "synthetic (rkmatch generator, on device)",
            "config": workload_config(per, sweep, world),
            "per_m_gbs": {str(m): (plans[m][1] - plans[m][0] + m - 1) / (per_m_ms[m] / 1e3) / 1e9
                          for m in sweep},
            "per_m_note": "per-length GB/s and the roofline come from a second pass of the "
                          "same steps (after a 1 s idle gap) with CUDA events around every "
                          "scan + emit; the headline steps run without events between the "
                          "launches, which would cost their programmatic-dependent-launch "
                          "overlap (~4%)",
            "matches_per_m": {str(m): int(host_counts[i, 0]) for i, m in enumerate(sweep)},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "traffic_per_m": traffic_per_m,
                         "traffic_source": tr.get("source") if tr else None,
                         # the same bytes over the headline steps' time (scans, emits and
                         # the gaps between them, no events in between)
                         "achieved_headline_steps": sum(alg) / (elapsed_ms / args.steps / 1e3) / 1e9,
                         "peak_kind": peak_kind, "kernel": "rk_scan_kernel<M>",
                         "algorithmic_bytes": "n + 8*matches per launch"},
            "sustained": sustained,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "e2e_per_call": e2e_call,
            "clocks": clk,
            "clocks_per_m_pass": clk_b.summary(),
            "gpu_launches": launches,
        }
        if comm is not None:
            line["exchange"] = {
                "api": ("rk_scan_sharded_batch_async (C ABI: one NCCL group all-gathering every "
                        "rank's counters and %d-offset slabs per pattern, ordered on the device; "
                        "no host round trip per step)" % args.slab) if batch_async[0] else
                       "rk_scan_sharded_batch (C ABI, NCCL allgather-v sized from the gathered "
                       "counts: a list was over the slab)",
                "nccl": comm.info()}
        print(json.dumps(line), flush=True)
    if comm is not None:
        comm.close()
    if world > 1:
        dist.destroy_process_group()


def run_c4(args, world, rank, dev):
    """BASELINE configs[3]: 16 GiB DNA, a sampled 32-byte pattern with copies planted
    across every 2/4/8-way shard cut, strong scaling: rank r holds its windows' bytes +
    the (m-1)-byte halo (rk_shard_range) and the global ordered list is returned to every
    rank by rk_scan_sharded."""
    import torch
    import torch.distributed as dist

    import paper_1810_01051_b200 as rk
    from paper_1810_01051_b200 import _lib, sharded

    n, m = args.c4_bytes, 32
    spec = rk.DnaSpec(SEED, n)
    a, b, blo, bhi = sharded.shard_range(n, m, world, rank)
    text = rk.generate_tensor(spec, device=f"cuda:{dev}", skip=blo, count=bhi - blo)
    x = sampled_offset(n, m)
    pat = rk.generate_tensor(spec, device=f"cuda:{dev}", skip=x, count=m).cpu().numpy().tobytes()
    cuts = sorted({sharded.shard_range(n, m, w, r)[0] for w in (2, 4, 8) for r in range(1, w)})
    plants = []
    for y in [c - m // 2 for c in cuts] + [n - m]:
        if not plants or y >= plants[-1] + m:
            plants.append(y)
    parr = torch.frombuffer(bytearray(pat), dtype=torch.uint8).to(f"cuda:{dev}")
    for y in plants:
        lo, hi = max(y, blo), min(y + m, bhi)
        if lo < hi:
            text[lo - blo: hi - blo] = parr[lo - y: hi - y]
    L = _lib.lib()
    comm = sharded.Communicator(device=dev)  # a 1-rank communicator at N = 1
    stream = torch.cuda.current_stream(dev)
    sptr = stream.cuda_stream
    out = torch.empty(1 << 20, dtype=torch.int64, device=f"cuda:{dev}")
    acounts = torch.zeros((1, 4), dtype=torch.int64, device=f"cuda:{dev}")
    res = {}
    use_async = [True]

    def step(_ev=None):
        if use_async[0]:
            # the exchange with no host round trip (one NCCL group: counters + a fixed slab
            # per rank, ordered on the device) -- a strong-scaling step is ~0.3 ms at N = 8
            comm.scan_batch_async(text, [pat], [(a, b)], blo, [out], acounts, slab=args.slab,
                                  stream=sptr)
        else:
            res["r"] = comm.scan(text, pat, a, b, blo, cap=out.numel(), out=out, stream=sptr)

    for _ in range(max(args.warmup, 3)):
        step()
    torch.cuda.synchronize()
    ac = acounts.cpu().numpy()[0]
    if ac[3]:  # a rank's list is over the slab: the synchronous exchange
        use_async[0] = False
        for _ in range(max(args.warmup, 3)):
            step()
        torch.cuda.synchronize()
        offs, k, coll, hits = res["r"]
    else:
        k, hits, coll = int(ac[0]), int(ac[1]), int(ac[2])
        offs = out[:k]
    got = set(offs.cpu().tolist())
    assert set(plants) <= got and hits == k + coll
    l0 = comm.ctx.launches
    elapsed_ms, clk = timed_steps(step, args.steps, stream, dev, world)
    launches = comm.ctx.launches - l0
    value = (n - m + 1) / (elapsed_ms / args.steps / 1e3) / 1e9
    peak, peak_kind = load_peaks()
    local_bytes = bhi - blo
    e2e = None
    if (args.e2e_steps or 0) > 0:
        host = text.cpu().pin_memory()
        t0 = time.perf_counter()
        for _ in range(args.e2e_steps):
            o2, k2, _, _ = comm.scan(host, pat, a, b, blo, cap=out.numel(), out=out, stream=sptr)
            o2.cpu()
        torch.cuda.synchronize()
        t_e = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device=f"cuda:{dev}")
        if world > 1:
            dist.all_reduce(t_e, op=dist.ReduceOp.MAX)
        e2e = {"value": (n - m + 1) / (float(t_e.item()) / args.e2e_steps) / 1e9, "unit": "GB/s",
               "h2d_bytes_per_step": local_bytes + m, "d2h_bytes_per_step": 8 * k + 32 * world,
               "steps": args.e2e_steps,
               "api": "rk_scan_sharded with this rank's pinned host shard (staged in 64 MiB "
                      "chunks overlapped with the scan) + the global list to host"}
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        import oracle

        threads = oracle.cpu_threads()
        sample = text[: 512 << 20].cpu().numpy()
        t0 = time.perf_counter()
        oracle.c_scan(sample, np.frombuffer(pat, dtype=np.uint8), workers=threads)
        dt = time.perf_counter() - t0
        cpu = {"value": sample.size / dt / 1e9, "unit": "GB/s", "cores": threads, "kind": "port",
               "sample": "512 MiB prefix of the C4 corpus, m = 32 (oracle C port of "
                         "_scan_range + search_parallel ranges)"}
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": elapsed_ms / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "u8",
            "data": "synthetic (rkmatch generator, on device)",
            "config": {"workload": "C4: 16 GiB synthetic DNA, 32-byte pattern, sharded with "
                                   "halo (BASELINE.json configs[3])",
                       "bytes_total": n, "m": m, "plants": len(plants),
                       "l2": "inputs larger than L2",
                       "parallelism": f"shard{world} (strong, rk_shard_range, (m-1)-byte halo)"},
            "matches": int(k), "collisions": int(coll),
            "roofline": {"bound": "hbm",
                         "achieved": (local_bytes + 8 * k) / (elapsed_ms / args.steps / 1e3) / 1e9,
                         "peak": peak, "unit": "GB/s", "peak_kind": peak_kind,
                         "kernel": "rk_scan_kernel<32> (+ emit + exchange)",
                         "algorithmic_bytes": "shard bytes + 8*matches per step"},
            "cpu_baseline": cpu, "e2e": e2e, "clocks": clk, "gpu_launches": launches,
            "exchange": {"api": ("rk_scan_sharded_batch_async (C ABI: one NCCL group, counters + "
                                 "a %d-offset slab per rank, ordered on the device)" % args.slab)
                                if use_async[0] else "rk_scan_sharded (C ABI, NCCL allgather-v)",
                         "nccl": comm.info()},
        }
        line["roofline"]["frac"] = line["roofline"]["achieved"] / peak
        print(json.dumps(line), flush=True)
    comm.close()
    if world > 1:
        dist.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
