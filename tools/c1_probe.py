import ctypes, time, sys, statistics
sys.path.insert(0, "/root/repo")
import numpy as np, torch
import paper_1810_01051_b200 as rk
from paper_1810_01051_b200 import _lib, _scan
spec = rk.DnaSpec(42, 1 << 20, bytes(range(32, 127)))
t = rk.generate_tensor(spec)
pat = rk.datagen.make_pattern(t, spec, 8, "sampled")
hx = rk.hash_full(pat); n = t.numel()
L = _lib.lib(); ctx = _lib.context()
out = torch.empty(4096, dtype=torch.int64, device="cuda")
p = np.frombuffer(pat, dtype=np.uint8)
mt, co, hh = _lib.u64ref(), _lib.u64ref(), _lib.u64ref()
s = torch.cuda.current_stream().cuda_stream
counts = torch.zeros(3, dtype=torch.int64, device="cuda")
def f_sync():
    _lib.check(L.rk_scan(ctx.handle, t.data_ptr(), n, p.ctypes.data, 8, hx, 0, n - 7, out.data_ptr(), 4096, ctypes.byref(mt), ctypes.byref(co), ctypes.byref(hh), s))
def f_async():
    _lib.check(L.rk_scan_async(ctx.handle, t.data_ptr(), n, p.ctypes.data, 8, hx, 0, n - 7, out.data_ptr(), 4096, 0, counts.data_ptr(), s))
def f_api():
    _scan.scan_counts(t, pat, hx, 0, n - 7)
for name, f in [("rk_scan sync", f_sync), ("scan_counts", f_api)]:
    for _ in range(20): f()
    ts = []
    for _ in range(200):
        a = time.perf_counter(); f(); ts.append(time.perf_counter() - a)
    print(name, "wall us median", round(statistics.median(ts) * 1e6, 1))
# device time of the async path
for _ in range(20): f_async()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); 
for _ in range(100): f_async()
e1.record(); torch.cuda.synchronize()
print("async back-to-back device us per scan", round(e0.elapsed_time(e1) * 1000 / 100, 1))
a = time.perf_counter()
for _ in range(100): f_async()
print("async enqueue host us per scan", round((time.perf_counter() - a) * 1e6 / 100, 1))
torch.cuda.synchronize()
