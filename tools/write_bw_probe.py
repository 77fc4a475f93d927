import torch, time
n = 1 << 28
out = torch.empty(n, dtype=torch.int64, device="cuda")
for _ in range(3): torch.arange(n, out=out); out.fill_(7)
torch.cuda.synchronize()
for name, f in (("arange", lambda: torch.arange(n, out=out)), ("fill", lambda: out.fill_(7)), ("zero", lambda: out.zero_())):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10): f()
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    print(name, "%.3f ms, %.2f TB/s write" % (ms, n * 8 / ms / 1e9))
