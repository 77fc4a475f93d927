"""Scan module -- the drop-in for rkmatch._scan (/root/reference/pkg/src/rkmatch/_scan.py).

Same three functions, same arguments and errors, backed by librkb200.so:

* ``as_u8(data)``        _scan.py:17-25 (also accepts 1-D uint8 torch tensors, CPU or CUDA)
* ``scan(text, pattern, hx, start, stop)``   _scan.py:53-68 -> (int64 offsets, collisions)
* ``window_hashes(text, m, start, stop)``    _scan.py:71-91 -> uint64 hashes

Host inputs go through ``rk_scan_host`` (chunked pinned staging into HBM overlapped with
the scan); CUDA tensors go straight to ``rk_scan`` on the current torch stream and give
CUDA results.  There is no CPU path.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib

_INITIAL_CAPACITY = 1 << 16  # offsets returned without a second pass (reference: 4096)


def _torch():
    import torch

    return torch


def _is_tensor(x) -> bool:
    try:
        import torch
    except ImportError:  # pragma: no cover
        return False
    return isinstance(x, torch.Tensor)


def as_u8(data):
    """View bytes-like input as a uint8 array without copying (_scan.py:17-25).

    bytes / bytearray / memoryview -> np.frombuffer; uint8 ndarray -> contiguous;
    1-D uint8 torch tensor -> contiguous tensor (kept on its device).  Anything else is
    a TypeError, as in the reference."""
    if isinstance(data, np.ndarray):
        if data.dtype != np.uint8:
            raise TypeError(f"expected uint8 array, got {data.dtype}")
        return np.ascontiguousarray(data).reshape(-1)
    if isinstance(data, (bytes, bytearray, memoryview)):
        return np.frombuffer(data, dtype=np.uint8)
    if _is_tensor(data):
        torch = _torch()
        if data.dtype != torch.uint8:
            raise TypeError(f"expected uint8 tensor, got {data.dtype}")
        return data.contiguous().reshape(-1)
    raise TypeError(f"expected bytes-like input, got {type(data).__name__}")


def _size(t) -> int:
    if _is_tensor(t):
        return int(t.numel())
    if isinstance(t, np.ndarray):
        return int(t.size)
    return len(t)


def _host_bytes(p) -> np.ndarray:
    if _is_tensor(p):
        return p.detach().to("cpu").contiguous().numpy()
    if isinstance(p, (bytes, bytearray, memoryview)):
        return np.frombuffer(p, dtype=np.uint8)
    if isinstance(p, np.ndarray):
        if p.dtype != np.uint8:
            raise TypeError(f"expected uint8 array, got {p.dtype}")
        return np.ascontiguousarray(p).reshape(-1)
    return np.frombuffer(bytes(p), dtype=np.uint8)


def _stream(dev: int) -> int:
    """Raw handle of the current CUDA stream of ``dev`` (what the C ABI takes).

    torch's own raw-stream accessor skips building a ``torch.cuda.Stream`` object
    (~2 us per call, a visible share of a launch-bound 1 MiB scan)."""
    torch = _torch()
    raw = getattr(torch._C, "_cuda_getCurrentRawStream", None)
    if raw is not None:
        return int(raw(dev))
    return torch.cuda.current_stream(dev).cuda_stream


def _device_of(t) -> int | None:
    if _is_tensor(t) and t.is_cuda:
        return t.device.index if t.device.index is not None else _torch().cuda.current_device()
    return None


def _ptr(a: np.ndarray) -> int:
    return a.ctypes.data if a.size else 0


def to_device(host: np.ndarray, dev: int):
    """A CUDA copy of a host uint8 array (read-only buffers such as ``bytes`` included):
    staged through a pinned buffer, so the upload is one DMA and no read-only numpy array
    is ever wrapped by a torch tensor."""
    torch = _torch()
    h = np.ascontiguousarray(host).reshape(-1)
    out = torch.empty(h.size, dtype=torch.uint8, device=f"cuda:{dev}")
    if h.size:
        pinned = torch.empty(h.size, dtype=torch.uint8, pin_memory=True)
        pinned.numpy()[:] = h
        out.copy_(pinned, non_blocking=True)
        torch.cuda.current_stream(dev).synchronize()  # the pinned buffer is freed after
    return out


def scan_counts(text, pattern, hx: int, start: int, stop: int, *, out_bias: int = 0,
                device: int | None = None):
    """Core call: (offsets, matches, collisions, hash_hits) for windows [start, stop).

    ``offsets`` is an int64 ndarray for host text and an int64 CUDA tensor for CUDA
    text, holding all matches in ascending order.  A host text is staged to ``device``
    (default: the current one)."""
    L = _lib.lib()
    p = _host_bytes(pattern)
    m = int(p.size)
    n = _size(text)
    hx = int(hx) & ((1 << 64) - 1)
    mt, co, hh = _lib.u64ref(), _lib.u64ref(), _lib.u64ref()
    dev = _device_of(text)
    if dev is None:
        t = _host_bytes(text)
        cap = max(0, min(stop - start, _INITIAL_CAPACITY))
        out = np.empty(max(cap, 1), dtype=np.int64)
        with _lib.acquire(device) as ctx:
            _lib.check(L.rk_scan_host(ctx.handle, _ptr(t), n, _ptr(p), m, hx, start, stop,
                                      out.ctypes.data, cap, ctypes.byref(mt), ctypes.byref(co),
                                      ctypes.byref(hh)))
            k = int(mt.value)
            if k > cap:
                out = np.empty(k, dtype=np.int64)
                _lib.check(L.rk_scan_host_fetch(ctx.handle, out.ctypes.data, 0, k))
        out = out[:k]
        if out_bias:
            out += out_bias
        return out, k, int(co.value), int(hh.value)

    torch = _torch()
    stream = _stream(dev)
    cap = max(0, min(stop - start, _INITIAL_CAPACITY))
    out = torch.empty(max(cap, 1), dtype=torch.int64, device=text.device)
    with _lib.acquire(dev) as ctx:
        _lib.check(L.rk_scan(ctx.handle, text.data_ptr(), n, _ptr(p), m, hx, start, stop,
                             out.data_ptr(), cap, ctypes.byref(mt), ctypes.byref(co),
                             ctypes.byref(hh), stream))
        k = int(mt.value)
        if k > cap:
            # the reference's overflow protocol (_scan.py:64-67) rescans with exact room;
            # here only the ordered emission runs again, from the scan's per-tile results
            out = torch.empty(k, dtype=torch.int64, device=text.device)
            _lib.check(L.rk_scan_fetch(ctx.handle, out.data_ptr(), k, stream))
    out = out[:k]
    if out_bias:
        out += out_bias
    return out, k, int(co.value), int(hh.value)


def scan(text, pattern, hx: int, start: int, stop: int):
    """Scan window offsets [start, stop); returns (offsets, collision count) (_scan.py:53-68)."""
    if stop <= start:
        if _device_of(text) is not None:
            torch = _torch()
            return torch.empty(0, dtype=torch.int64, device=text.device), 0
        return np.empty(0, dtype=np.int64), 0
    offsets, _, collisions, _ = scan_counts(text, pattern, hx, start, stop)
    return offsets, collisions


def scan_bitmap(text, pattern, hx: int, start: int, stop: int, *, packed: bool = False):
    """Match bitmap of windows [start, stop) computed on the device (rk_scan_bitmap):
    element i is True iff window start+i matches -- MatchResult.to_bitmap
    (matcher.py:36-42) without materialising offsets (1 bit per window instead of 8 bytes
    per match).  Returns (bitmap, matches, collisions, hash_hits); the bitmap is a bool
    CUDA tensor for CUDA text, a bool ndarray for host text, or the packed uint32 words
    (bit i%32 of word i/32) with packed=True."""
    torch = _torch()
    L = _lib.lib()
    p = _host_bytes(pattern)
    m = int(p.size)
    n = _size(text)
    if m == 0:
        raise ValueError("empty pattern")
    count = max(stop - start, 0)
    dev = _device_of(text)
    on_host = dev is None
    if on_host:
        dev = _lib.default_device()
        t = to_device(_host_bytes(text), dev)
    else:
        t = text
    words = torch.zeros(max((count + 31) // 32, 1), dtype=torch.int32, device=t.device)
    counts = torch.zeros(3, dtype=torch.int64, device=t.device)
    stream = _stream(dev)
    with _lib.acquire(dev) as ctx:
        _lib.check(L.rk_scan_bitmap(ctx.handle, t.data_ptr() if n else 0, n, _ptr(p), m,
                                    int(hx) & ((1 << 64) - 1), start, max(stop, start),
                                    words.data_ptr(), counts.data_ptr(), stream))
    mt, hh, co = (int(v) for v in counts.cpu().tolist())
    if packed:
        return (words.cpu().numpy().view(np.uint32) if on_host else words), mt, co, hh
    if on_host:
        bits = np.unpackbits(words.cpu().numpy().view(np.uint8), bitorder="little")[:count]
        return bits.astype(bool), mt, co, hh
    shifts = torch.arange(32, device=t.device, dtype=torch.int32)
    bits = ((words.unsqueeze(1) >> shifts) & 1).reshape(-1)[:count].bool()
    return bits, mt, co, hh


def window_hashes(text, m: int, start: int, stop: int):
    """uint64 hashes of every window [x, x+m), x in [start, stop) (_scan.py:71-91)."""
    if m < 1:
        raise ValueError("window length must be >= 1")
    n = _size(text)
    if start == stop:
        if _device_of(text) is not None:
            torch = _torch()
            return torch.empty(0, dtype=torch.uint64, device=text.device)
        return np.empty(0, dtype=np.uint64)
    if start < 0 or stop < start or stop - 1 + m > n:
        raise ValueError(
            f"window range [{start}, {stop}) of length {m} out of bounds "
            f"for text of length {n}"
        )
    torch = _torch()
    dev = _device_of(text)
    on_host = dev is None
    if on_host:
        dev = _lib.default_device()
        t = to_device(_host_bytes(text), dev)
    else:
        t = text
    out = torch.empty(stop - start, dtype=torch.uint64, device=t.device)
    stream = _stream(dev)
    with _lib.acquire(dev) as ctx:
        _lib.check(_lib.lib().rk_window_hashes(ctx.handle, t.data_ptr(), n, m, start, stop,
                                               out.data_ptr(), stream))
    if on_host:
        return out.cpu().numpy()
    return out
