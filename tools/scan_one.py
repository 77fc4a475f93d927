"""Device-timed single-pattern scans of the C2 corpus for chosen pattern lengths (a
profiling driver: `ncu -k regex:rk_scan_kernel ... python tools/scan_one.py --m 4`).

    python tools/scan_one.py --m 4,8,16 [--bytes 1GiB] [--reps 5] [--lib variant.so]

--lib times a variant library built with RK_DEFINES / RK_LIB_OUT (paper_1810_01051_b200/_build.py)
instead of the package's librkb200.so (A/B experiments).
"""

import argparse
import os
import statistics
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch

    import paper_1810_01051_b200 as rk
    from paper_1810_01051_b200 import _lib

    ap = argparse.ArgumentParser()
    ap.add_argument("--lib", default=None)
    ap.add_argument("--m", default="4")
    ap.add_argument("--bytes", type=int, default=1 << 30)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--source", default="sampled", choices=("sampled", "generated"))
    ap.add_argument("--fill", default=None, help="text of one repeated byte (C5: --fill a)")
    args = ap.parse_args()
    if args.lib:
        from pathlib import Path

        _lib.LIB_PATH = Path(args.lib).resolve()
    n = args.bytes
    spec = rk.DnaSpec(42, n, bytes(range(32, 127)))
    if args.fill:
        t = torch.full((n,), ord(args.fill), dtype=torch.uint8, device="cuda")
    else:
        t = rk.generate_tensor(spec)
    ctx = _lib.context()
    L = _lib.lib()
    s = torch.cuda.current_stream()
    counts = torch.zeros(3, dtype=torch.int64, device="cuda")
    out = torch.empty(n if args.fill else 1 << 20, dtype=torch.int64, device="cuda")
    for m in [int(x) for x in args.m.split(",")]:
        if args.fill:
            pat = np.frombuffer(args.fill.encode() * m, dtype=np.uint8)
        else:
            pat = np.frombuffer(rk.datagen.make_pattern(t, spec, m, args.source), dtype=np.uint8)
        hx = rk.hash_full(pat.tobytes())
        times = []
        for _ in range(args.reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            _lib.check(L.rk_scan_async(ctx.handle, t.data_ptr(), n, pat.ctypes.data, m, hx, 0,
                                       n - m + 1, out.data_ptr(), out.numel(), 0,
                                       counts.data_ptr(), s.cuda_stream))
            e1.record(s)
            e1.synchronize()
            times.append(e0.elapsed_time(e1))
        ms = statistics.median(times)
        c = counts.tolist()
        print(f"{args.lib or 'lib'} m={m} ms={ms:.4f} GB/s={n / ms / 1e6:.1f} matches={c[0]} hits={c[1]} "
              f"collisions={c[2]}")


if __name__ == "__main__":
    main()
