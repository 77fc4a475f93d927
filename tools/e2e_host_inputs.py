"""End-to-end search_sequential on a 1 GiB host text: bytes, ndarray and pinned tensor
(pageable inputs go through the multi-threaded pinned staging ring)."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_1810_01051_b200 as rk  # noqa: E402

spec = rk.DnaSpec(42, 1 << 30, bytes(range(32, 127)))
t = rk.generate_tensor(spec)
host = t.cpu().numpy()
b = host.tobytes()
pat = b[12345:12361]
for name, x in [("bytes", b), ("ndarray", host), ("pinned", t.cpu().pin_memory())]:
    rk.search_sequential(x, pat)
    t0 = time.perf_counter()
    r = rk.search_sequential(x, pat)
    dt = time.perf_counter() - t0
    print(name, len(r.offsets), f"{(1 << 30) / dt / 1e9:.1f} GB/s")
