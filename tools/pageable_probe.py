import time, os, sys, numpy as np, torch
sys.path.insert(0, os.getcwd())
from paper_1810_01051_b200 import _lib
if len(sys.argv) > 1: _lib.LIB_PATH = __import__("pathlib").Path(sys.argv[1]).resolve()
import paper_1810_01051_b200 as rk
n = 1 << 30
t = rk.generate_tensor(rk.DnaSpec(42, n, bytes(range(32, 127))))
host_bytes = t.cpu().numpy().tobytes()
pinned = t.cpu().pin_memory()
pats = [host_bytes[x:x + m] for x, m in ((1000, 4), (2000, 8), (3000, 16), (4000, 32), (5000, 64), (6000, 128), (7000, 256), (8000, 512), (9000, 1024))]
for name, src in (("pageable", host_bytes), ("pinned", pinned.numpy())):
    rk.search_each(src, pats)
    t0 = time.perf_counter(); rk.search_each(src, pats); dt = time.perf_counter() - t0
    t1 = time.perf_counter(); rk.search_sequential(src, pats[1]); dt1 = time.perf_counter() - t1
    print(name, os.environ.get("RKB200_COPY_THREADS", "8"), "each: %.1f GB/s text (%.1f ms)" % (n / dt / 1e9, dt * 1e3), "single: %.1f GB/s" % (n / dt1 / 1e9))
ts = []
for _ in range(6):
    t1 = time.perf_counter(); rk.search_sequential(host_bytes, pats[1]); ts.append(n / (time.perf_counter() - t1) / 1e9)
print("single x6:", " ".join("%.1f" % x for x in ts))
ts = []
for _ in range(6):
    t1 = time.perf_counter(); rk.search_each(host_bytes, pats); ts.append(n / (time.perf_counter() - t1) / 1e9)
print("each x6:", " ".join("%.1f" % x for x in ts))
