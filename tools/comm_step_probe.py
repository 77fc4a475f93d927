"""Per-step time of the C2 sweep through plain rk_scan_async, the synchronous sharded batch
(rk_scan_sharded_batch) and the asynchronous one (rk_scan_sharded_batch_async), one rank."""
import sys, time
sys.path.insert(0, "/root/repo")
import torch
import paper_1810_01051_b200 as rk
from paper_1810_01051_b200 import sharded, _lib, _scan
import numpy as np
ASCII = bytes(range(32, 127))
n = 1 << 30
spec = rk.DnaSpec(42, n, ASCII)
t = rk.generate_tensor(spec)
sweep = [4, 8, 16, 32, 64, 128, 256, 512, 1024]
pats = [t[1000 + 7919 * i: 1000 + 7919 * i + m].cpu().numpy().tobytes() for i, m in enumerate(sweep)]
comm = sharded.Communicator(device=0)
outs = [torch.empty(1 << 22, dtype=torch.int64, device="cuda") for _ in sweep]
s = torch.cuda.current_stream()
def step_comm():
    comm.scan_batch(t, pats, [(0, n - m + 1) for m in sweep], 0, outs, stream=s.cuda_stream)
acounts = torch.zeros((9, 4), dtype=torch.int64, device="cuda")
def step_async():
    comm.scan_batch_async(t, pats, [(0, n - m + 1) for m in sweep], 0, outs, acounts, stream=s.cuda_stream)
ctx = _lib.context(0); L = _lib.lib()
counts = torch.zeros((9, 3), dtype=torch.int64, device="cuda")
pb = [np.frombuffer(p, dtype=np.uint8) for p in pats]
def step_plain():
    for i, m in enumerate(sweep):
        _lib.check(L.rk_scan_async(ctx.handle, t.data_ptr(), n, pb[i].ctypes.data, m, rk.hash_full(pats[i]), 0, n - m + 1, outs[i].data_ptr(), 1 << 22, 0, counts[i].data_ptr(), s.cuda_stream))
for f, name in ((step_plain, "plain"), (step_comm, "comm"), (step_async, "async")) * 3:
    for _ in range(3): f()
    torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record(s)
    for _ in range(20): f()
    b.record(s); torch.cuda.synchronize()
    print(name, round(a.elapsed_time(b) / 20, 4), "ms/step")
