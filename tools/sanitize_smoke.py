"""Small end-to-end exercise of every kernel for compute-sanitizer (memcheck/racecheck):
    compute-sanitizer --tool memcheck python tools/sanitize_smoke.py
Edge cases on purpose: unaligned views, tiny texts, ranges, dense matches, m >= 65."""

import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import paper_1810_01051_b200 as rk  # noqa: E402
from paper_1810_01051_b200 import _scan  # noqa: E402


def main():
    rng = np.random.default_rng(1)
    base = torch.from_numpy(rng.integers(0, 3, 300000, dtype=np.uint8)).cuda()
    for shift in (0, 1, 31):
        t = base[shift : shift + 200000 - shift]
        for m in (1, 4, 5, 6, 8, 12, 16, 20, 31, 32, 40, 100):
            pat = t[777 : 777 + m].cpu().numpy().tobytes()
            rk.search_sequential(t, pat)
            _scan.scan(t, pat, rk.hash_full(pat), 5, 150000)
            _scan.scan_bitmap(t, pat, rk.hash_full(pat), 3, 190000)
    for n in (1, 2, 5, 31, 33, 1000, 100000):
        t = torch.full((n,), 97, dtype=torch.uint8, device="cuda")
        for m in (1, 2, 4, 6, 8, 33):
            if m <= n:
                rk.search_sequential(t, b"a" * m)
                _scan.scan_bitmap(t, b"a" * m, rk.hash_full(b"a" * m), 0, n - m + 1)
    host = rng.integers(0, 4, 100000, dtype=np.uint8)
    rk.search_sequential(host.tobytes(), host[10:30].tobytes())
    pats = [host[x : x + m].tobytes() for m in (3, 9, 16, 40) for x in (0, 50, 99000)]
    rk.search_multi(host.tobytes(), pats)
    rk.search_multi(base[1:70001], [base[100:116].cpu().numpy().tobytes()])
    for m in (4, 5, 6):  # anchored q-gram tiny kernel, staged and edge tiles
        rk.search_multi(base[3:150003], [base[x : x + m].cpu().numpy().tobytes() for x in (0, 9, 4093)])
    _scan.window_hashes(host, 7, 0, 1000)
    rk.generate(rk.DnaSpec(5, 12345))
    torch.cuda.synchronize()
    print("sanitize smoke ok")


if __name__ == "__main__":
    main()
