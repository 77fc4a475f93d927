"""Repeats small-cap scans + re-emits (tests/test_gpu_capi_state.py's shapes) and counts
mismatching match counts / offset lists: a race check for the emit (--lib: a variant)."""
import argparse
import ctypes
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--lib", default=None)
    ap.add_argument("--reps", type=int, default=30)
    args = ap.parse_args()
    from paper_1810_01051_b200 import _lib
    if args.lib:
        _lib.LIB_PATH = Path(args.lib).resolve()
    import torch

    import paper_1810_01051_b200 as rk
    import oracle
    from paper_1810_01051_b200 import _scan

    spec = rk.DnaSpec(7, 1 << 22, b"ab")
    text = rk.generate_tensor(spec, device="cuda")
    host = text.cpu().numpy()
    L = _lib.lib()
    ctx = _lib.context(0)
    s = _scan._stream(0)
    bad = 0
    exps = {}
    for pat in (b"abba", b"aaaaaaaaaaaa", b"ab"):
        exps[pat] = oracle.c_scan(host, np.frombuffer(pat, dtype=np.uint8))[0]
    for r in range(args.reps):
        for pat, exp in exps.items():
            p = np.frombuffer(pat, dtype=np.uint8)
            mt, co, hh = _lib.u64ref(), _lib.u64ref(), _lib.u64ref()
            small = torch.empty(5, dtype=torch.int64, device="cuda")
            _lib.check(L.rk_scan(ctx.handle, text.data_ptr(), text.numel(), p.ctypes.data,
                                 len(pat), rk.hash_full(pat), 0, text.numel() - len(pat) + 1,
                                 small.data_ptr(), 5, ctypes.byref(mt), ctypes.byref(co),
                                 ctypes.byref(hh), s))
            k = int(mt.value)
            big = torch.empty(max(k, 1), dtype=torch.int64, device="cuda")
            _lib.check(L.rk_scan_fetch(ctx.handle, big.data_ptr(), k, s))
            ok = k == len(exp) and np.array_equal(big[:k].cpu().numpy(), exp)
            if not ok:
                bad += 1
                print("mismatch", r, pat, k, len(exp), flush=True)
    print(f"lib={args.lib} bad={bad} of {args.reps * 3}")


if __name__ == "__main__":
    main()
