import sys, time, os
sys.path.insert(0, os.getcwd())
import torch, ctypes
import paper_1810_01051_b200 as rk
from paper_1810_01051_b200 import _scan, _lib
ASCII = bytes(range(32, 127))
spec = rk.DnaSpec(42, 1 << 20, ASCII)
t = rk.generate_tensor(spec)
pat = rk.datagen.make_pattern(t, spec, 8, "sampled")
hx = rk.hash_full(pat)
n = t.numel()
for _ in range(20): _scan.scan_counts(t, pat, hx, 0, n - 7)
torch.cuda.synchronize()
R = 200
t0 = time.perf_counter()
for _ in range(R): _scan.scan_counts(t, pat, hx, 0, n - 7)
t1 = time.perf_counter()
print("scan_counts host wall us/call", (t1 - t0) / R * 1e6)
# device-only: async enqueue R times, events
L = _lib.lib(); ctx = _lib.context(0)
s = torch.cuda.current_stream()
out = torch.empty(4096, dtype=torch.int64, device="cuda")
p = (ctypes.c_uint8 * 8).from_buffer_copy(bytes(pat))
a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
a.record(s)
for _ in range(R):
    L.rk_scan_async(ctx.handle, t.data_ptr(), n, p, 8, hx, 0, n - 7, out.data_ptr(), 4096, 0, None, s.cuda_stream)
b.record(s); torch.cuda.synchronize()
print("rk_scan_async back-to-back device us/scan", a.elapsed_time(b) / R * 1e3)
t0 = time.perf_counter()
mt, co, hh = _lib.u64ref(), _lib.u64ref(), _lib.u64ref()
for _ in range(R):
    L.rk_scan(ctx.handle, t.data_ptr(), n, p, 8, hx, 0, n - 7, out.data_ptr(), 4096, ctypes.byref(mt), ctypes.byref(co), ctypes.byref(hh), s.cuda_stream)
t1 = time.perf_counter()
print("rk_scan sync host wall us/call", (t1 - t0) / R * 1e6)
