#!/usr/bin/env python
"""Device-timed measurements of the other BASELINE.json configs on one B200 (bench.py
carries the headline, configs[1]).  Prints one JSON line per config.

  C1  single 8-byte pattern over 1 MiB printable ASCII (L2-resident, launch-bound)
  C3  1,024 equal-length (m=16) patterns over 4 GiB printable ASCII (search_multi)
  C4  16 GiB DNA, 32-byte pattern with copies planted across shard boundaries (N=1)
  C5  all 'a', pattern 'aaaa' (every window matches; write-bound), 256 MiB

    python bench_configs.py [--only C3,C5] [--reps 5]
"""

from __future__ import annotations

import argparse
import ctypes
import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

ASCII = bytes(range(32, 127))


def timed(fn, reps, stream):
    import torch

    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        fn()
        b.record(stream)
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return sorted(ts)[len(ts) // 2]


def c1(reps):
    import torch

    import paper_1810_01051_b200 as rk
    from paper_1810_01051_b200 import _scan

    spec = rk.DnaSpec(42, 1 << 20, ASCII)
    t = rk.generate_tensor(spec)
    pat = rk.datagen.make_pattern(t, spec, 8, "sampled")
    hx = rk.hash_full(pat)
    s = torch.cuda.current_stream()
    ms = timed(lambda: _scan.scan_counts(t, pat, hx, 0, t.numel() - 7), reps, s)
    offs, k, coll, hits = _scan.scan_counts(t, pat, hx, 0, t.numel() - 7)
    return {"config": "C1", "bytes": t.numel(), "m": 8, "ms": ms,
            "GBps": t.numel() / ms / 1e6, "matches": k, "collisions": coll,
            "note": "includes the host round trip of the synchronous rk_scan (counters written to mapped pinned memory) and the Python wrapper"}


def c3(reps, n=4 << 30, P=1024, m=16, alphabet=None, tag="C3"):
    import torch

    import paper_1810_01051_b200 as rk
    from paper_1810_01051_b200 import _lib, datagen

    alphabet = ASCII if alphabet is None else alphabet
    spec = rk.DnaSpec(43, n, alphabet)
    t = rk.generate_tensor(spec)
    pats = []
    state = 43
    for _ in range(P // 2):
        draw, state = datagen.splitmix64(state)
        x = draw % (n - m + 1)
        pats.append(t[x: x + m].cpu().numpy().tobytes())
    for j in range(P - P // 2):
        pats.append(rk.generate(rk.DnaSpec((43 ^ 0x5DEECE66D) + j, m, alphabet)))
    ps = rk.PatternSet(pats)
    flat = np.frombuffer(b"".join(ps.patterns), dtype=np.uint8)
    hashes = np.array([rk.hash_full(p) for p in ps.patterns], dtype=np.uint64)
    ctx = _lib.context()
    L = _lib.lib()
    cap = 1 << 20
    off = torch.empty(cap, dtype=torch.int64, device="cuda")
    idx = torch.empty(cap, dtype=torch.int32, device="cuda")
    pairs = _lib.u64ref()
    s = torch.cuda.current_stream()

    def run():
        _lib.check(L.rk_multi_scan(ctx.handle, t.data_ptr(), n, flat.ctypes.data, len(ps), m,
                                   hashes.ctypes.data, off.data_ptr(), idx.data_ptr(), cap,
                                   ctypes.byref(pairs), s.cuda_stream))

    ms = timed(run, reps, s)
    return {"config": tag, "bytes": n, "patterns": len(ps), "m": m, "ms": ms,
            "GBps": n / ms / 1e6, "pairs": int(pairs.value),
            "note": "rk_multi_scan incl. table build + host ordering of the pairs"}


def c3_mixed(reps, n=4 << 30, P=1024):
    """C3's corpus and shape with mixed lengths 8..71 (64 distinct -> 4 sweeps of 16
    lengths) through rk_multi_scan_mixed (not a BASELINE config)."""
    import torch

    import paper_1810_01051_b200 as rk
    from paper_1810_01051_b200 import _lib, datagen

    spec = rk.DnaSpec(43, n, ASCII)
    t = rk.generate_tensor(spec)
    pats = []
    state = 43
    for i in range(P):
        m = 8 + i % 64
        draw, state = datagen.splitmix64(state)
        x = draw % (n - m + 1)
        pats.append(t[x: x + m].cpu().numpy().tobytes())
    ps = rk.PatternSet(pats)
    flat = np.frombuffer(b"".join(ps.patterns), dtype=np.uint8)
    lengths = np.array([len(p) for p in ps.patterns], dtype=np.uint32)
    hashes = np.array([rk.hash_full(p) for p in ps.patterns], dtype=np.uint64)
    ctx = _lib.context()
    L = _lib.lib()
    cap = 1 << 20
    off = torch.empty(cap, dtype=torch.int64, device="cuda")
    idx = torch.empty(cap, dtype=torch.int32, device="cuda")
    pairs = _lib.u64ref()
    s = torch.cuda.current_stream()

    def run():
        _lib.check(L.rk_multi_scan_mixed(ctx.handle, t.data_ptr(), n, flat.ctypes.data,
                                         lengths.ctypes.data, len(ps), hashes.ctypes.data,
                                         off.data_ptr(), idx.data_ptr(), cap, ctypes.byref(pairs),
                                         s.cuda_stream))

    before = ctx.launches
    run()
    sweeps = ctx.launches - before
    ms = timed(run, reps, s)
    return {"config": "C3mixed", "bytes": n, "patterns": len(ps), "lengths": "8..71",
            "sweeps": sweeps, "ms": ms, "GBps": n / ms / 1e6, "pairs": int(pairs.value),
            "note": "rk_multi_scan_mixed incl. table build + host ordering of the pairs"}


def c3_dense(reps, n=64 << 20, lengths=(4, 5, 6)):
    """Dense multi-pattern output: all 'a' with {'aaaa', 'aaaaa', 'aaaaaa'} (every window of
    every length matches: ~3n (offset, index) pairs through rk_multi_scan_mixed, the ordered
    device sort included).  Parity: each pattern's list is range(n - m + 1)."""
    import torch

    import paper_1810_01051_b200 as rk
    from paper_1810_01051_b200 import _lib

    t = torch.full((n,), 97, dtype=torch.uint8, device="cuda")
    pats = [b"a" * m for m in lengths]
    flat = np.frombuffer(b"".join(pats), dtype=np.uint8)
    lens = np.array(lengths, dtype=np.uint32)
    hashes = np.array([rk.hash_full(p) for p in pats], dtype=np.uint64)
    total = sum(n - m + 1 for m in lengths)
    off = torch.empty(total, dtype=torch.int64, device="cuda")
    idx = torch.empty(total, dtype=torch.int32, device="cuda")
    pairs = _lib.u64ref()
    ctx = _lib.context()
    L = _lib.lib()
    s = torch.cuda.current_stream()

    def run():
        _lib.check(L.rk_multi_scan_mixed(ctx.handle, t.data_ptr(), n, flat.ctypes.data,
                                         lens.ctypes.data, len(pats), hashes.ctypes.data,
                                         off.data_ptr(), idx.data_ptr(), total,
                                         ctypes.byref(pairs), s.cuda_stream))

    before = ctx.launches
    run()
    sweeps = ctx.launches - before
    ms = timed(run, reps, s)
    assert int(pairs.value) == total
    at = 0
    for i, m in enumerate(lengths):
        k = n - m + 1
        assert torch.equal(idx[at:at + k], torch.full((k,), i, dtype=torch.int32, device="cuda"))
        assert torch.equal(off[at:at + k], torch.arange(k, device="cuda"))
        at += k
    return {"config": "C3dense", "bytes": n, "lengths": list(lengths), "pairs": total,
            "launches": sweeps, "ms": ms, "GBps_text": n / ms / 1e6,
            "Mpairs_per_s": total / ms / 1e3,
            "note": "all 'a', every window of every length matches; parity checked on device"}


def c4(reps, n=16 << 30, m=32):
    import torch

    import paper_1810_01051_b200 as rk
    from paper_1810_01051_b200 import _scan

    spec = rk.DnaSpec(42, n)
    t = rk.generate_tensor(spec)
    pat = rk.datagen.make_pattern(t, spec, m, "sampled")
    p = torch.frombuffer(bytearray(pat), dtype=torch.uint8).cuda()
    for g in range(1, 8):
        x = g * (n // 8) - 16
        t[x: x + m] = p
    hx = rk.hash_full(pat)
    s = torch.cuda.current_stream()
    ms = timed(lambda: _scan.scan_counts(t, pat, hx, 0, n - m + 1), reps, s)
    offs, k, coll, hits = _scan.scan_counts(t, pat, hx, 0, n - m + 1)
    return {"config": "C4", "bytes": n, "m": m, "ms": ms, "GBps": n / ms / 1e6, "matches": k,
            "collisions": coll, "gpus": 1}


def c5(reps, n=1 << 28):
    import torch

    import paper_1810_01051_b200 as rk
    from paper_1810_01051_b200 import _lib

    t = torch.full((n,), 97, dtype=torch.uint8, device="cuda")
    out = torch.empty(n, dtype=torch.int64, device="cuda")
    counts = torch.zeros(3, dtype=torch.int64, device="cuda")
    pat = np.frombuffer(b"aaaa", dtype=np.uint8)
    ctx = _lib.context()
    L = _lib.lib()
    s = torch.cuda.current_stream()

    def run():
        _lib.check(L.rk_scan_async(ctx.handle, t.data_ptr(), n, pat.ctypes.data, 4,
                                   rk.hash_full(b"aaaa"), 0, n - 3, out.data_ptr(), n, 0,
                                   counts.data_ptr(), s.cuda_stream))

    ms = timed(run, reps, s)
    k = int(counts[0].item())
    assert k == n - 3
    assert torch.equal(out[: n - 3], torch.arange(n - 3, device="cuda"))
    alg = n + 8 * (n - 3)
    return {"config": "C5", "bytes": n, "m": 4, "ms": ms, "GBps_text": n / ms / 1e6,
            "GBps_algorithmic": alg / ms / 1e6, "matches": k}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default="C1,C3,C4,C5")
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--lib", default=None, help="time a variant library (A/B experiments)")
    args = ap.parse_args()
    if args.lib:
        from pathlib import Path

        from paper_1810_01051_b200 import _lib

        _lib.LIB_PATH = Path(args.lib).resolve()
    fns = {"C1": c1, "C3": c3, "C4": c4, "C5": c5,
           # not a BASELINE config: C3's shape over DNA (low-entropy q-grams)
           "C3dna": lambda r: c3(r, m=32, alphabet=b"ACGT", tag="C3dna"),
           "C3mixed": c3_mixed,
           "C3dense": c3_dense,
           "C3short6": lambda r: c3(r, m=6, tag="C3short6"),
           "C3short": lambda r: c3(r, m=5, tag="C3short"),
           "C3short4": lambda r: c3(r, m=4, tag="C3short4")}
    for name in args.only.split(","):
        t0 = time.time()
        r = fns[name](args.reps)
        r["wall_s"] = round(time.time() - t0, 1)
        if args.lib:
            r["lib"] = args.lib
        print(json.dumps(r), flush=True)


if __name__ == "__main__":
    main()
