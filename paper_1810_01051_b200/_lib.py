"""ctypes binding of librkb200.so (include/rkb200.h) and per-device contexts.

There is no fallback: if the library is missing, or no sm_100 device is visible, every
search entry point raises.  (The CPU oracle under ``oracle/`` is test infrastructure and
is never imported from here.)
"""

from __future__ import annotations

import atexit
import ctypes
import os
import threading
from pathlib import Path

LIB_PATH = Path(__file__).resolve().parent / "librkb200.so"

RK_OK, RK_EINVAL, RK_ECUDA, RK_ENCCL = 0, 1, 2, 3
COMM_ID_BYTES = 128
MULTI_MAX_PATTERNS = 4096
BATCH_MAX_PATTERNS = 64

# every symbol include/rkb200.h declares (checked by tests/test_capi.py)
EXPORTS = (
    "rk_version", "rk_last_error", "rk_device_count", "rk_ctx_create", "rk_ctx_destroy",
    "rk_scan", "rk_scan_async", "rk_scan_result", "rk_scan_bitmap", "rk_scan_host",
    "rk_scan_host_fetch", "rk_scan_fetch", "rk_scan_host_batch",
    "rk_multi_scan", "rk_multi_scan_mixed", "rk_window_hashes", "rk_generate", "rk_launch_count",
    "rk_comm_get_unique_id", "rk_comm_init", "rk_comm_destroy", "rk_comm_info", "rk_shard_range",
    "rk_scan_sharded", "rk_comm_fetch", "rk_multi_scan_sharded", "rk_scan_sharded_batch",
    "rk_scan_sharded_batch_async",
)

_lib = None
_lib_lock = threading.Lock()


def _declare(lib: ctypes.CDLL) -> None:
    u8p = ctypes.c_void_p
    u64 = ctypes.c_uint64
    u32 = ctypes.c_uint32
    i64 = ctypes.c_int64
    pu64 = ctypes.POINTER(ctypes.c_uint64)
    vp = ctypes.c_void_p
    ci = ctypes.c_int
    lib.rk_version.restype = ctypes.c_char_p
    lib.rk_version.argtypes = []
    lib.rk_last_error.restype = ctypes.c_char_p
    lib.rk_last_error.argtypes = []
    lib.rk_device_count.restype = ci
    lib.rk_device_count.argtypes = []
    lib.rk_ctx_create.restype = ci
    lib.rk_ctx_create.argtypes = [ci, ctypes.POINTER(vp)]
    lib.rk_ctx_destroy.restype = ci
    lib.rk_ctx_destroy.argtypes = [vp]
    lib.rk_scan.restype = ci
    lib.rk_scan.argtypes = [vp, u8p, u64, u8p, u32, u64, u64, u64, vp, u64, pu64, pu64, pu64, vp]
    lib.rk_scan_async.restype = ci
    lib.rk_scan_async.argtypes = [vp, u8p, u64, u8p, u32, u64, u64, u64, vp, u64, i64, vp, vp]
    lib.rk_scan_bitmap.restype = ci
    lib.rk_scan_bitmap.argtypes = [vp, u8p, u64, u8p, u32, u64, u64, u64, vp, vp, vp]
    lib.rk_scan_result.restype = ci
    lib.rk_scan_result.argtypes = [vp, pu64, pu64, pu64, vp]
    lib.rk_scan_host.restype = ci
    lib.rk_scan_host.argtypes = [vp, u8p, u64, u8p, u32, u64, u64, u64, vp, u64, pu64, pu64, pu64]
    lib.rk_scan_host_batch.restype = ci
    lib.rk_scan_host_batch.argtypes = [vp, u8p, u64, u8p, vp, vp, ctypes.c_uint32, vp, u64, vp,
                                       vp, vp]
    lib.rk_scan_host_fetch.restype = ci
    lib.rk_scan_host_fetch.argtypes = [vp, vp, u64, u64]
    lib.rk_scan_fetch.restype = ci
    lib.rk_scan_fetch.argtypes = [vp, vp, u64, vp]
    lib.rk_multi_scan.restype = ci
    lib.rk_multi_scan.argtypes = [vp, u8p, u64, u8p, u32, u32, vp, vp, vp, u64, pu64, vp]
    lib.rk_multi_scan_mixed.restype = ci
    lib.rk_multi_scan_mixed.argtypes = [vp, u8p, u64, u8p, vp, u32, vp, vp, vp, u64, pu64, vp]
    lib.rk_window_hashes.restype = ci
    lib.rk_window_hashes.argtypes = [vp, u8p, u64, u32, u64, u64, vp, vp]
    lib.rk_generate.restype = ci
    lib.rk_generate.argtypes = [vp, vp, u64, u64, u64, u8p, u32, vp]
    lib.rk_launch_count.restype = u64
    lib.rk_launch_count.argtypes = [vp]
    pi = ctypes.POINTER(ci)
    lib.rk_comm_get_unique_id.restype = ci
    lib.rk_comm_get_unique_id.argtypes = [vp]
    lib.rk_comm_init.restype = ci
    lib.rk_comm_init.argtypes = [vp, vp, ci, ci, ctypes.POINTER(vp)]
    lib.rk_comm_destroy.restype = ci
    lib.rk_comm_destroy.argtypes = [vp]
    lib.rk_comm_info.restype = ci
    lib.rk_comm_info.argtypes = [vp, pi, pi, pi]
    lib.rk_shard_range.restype = ci
    lib.rk_shard_range.argtypes = [u64, u32, ci, ci, pu64, pu64, pu64, pu64]
    lib.rk_scan_sharded_batch.restype = ci
    lib.rk_scan_sharded_batch.argtypes = [vp, u8p, u64, u64, u8p, vp, vp, u32, vp, vp, vp, vp, vp,
                                          vp, vp, vp]
    lib.rk_scan_sharded_batch_async.restype = ci
    lib.rk_scan_sharded_batch_async.argtypes = [vp, u8p, u64, u64, u8p, vp, vp, u32, vp, vp, vp,
                                                vp, u64, vp, vp]
    lib.rk_multi_scan_sharded.restype = ci
    lib.rk_multi_scan_sharded.argtypes = [vp, u8p, u64, u64, u64, u8p, vp, u32, vp, u64, u64, vp,
                                          vp, u64, pu64, vp]
    lib.rk_comm_fetch.restype = ci
    lib.rk_comm_fetch.argtypes = [vp, vp, u64, u64, vp]
    lib.rk_scan_sharded.restype = ci
    lib.rk_scan_sharded.argtypes = [vp, u8p, u64, u64, u8p, u32, u64, u64, u64, vp, u64, pu64,
                                    pu64, pu64, vp]


def lib() -> ctypes.CDLL:
    """The loaded library (raises if it has not been built)."""
    global _lib
    if _lib is not None:
        return _lib
    with _lib_lock:
        if _lib is None:
            if not LIB_PATH.exists():
                raise RuntimeError(
                    f"{LIB_PATH} is missing: build it with `python -m paper_1810_01051_b200._build`"
                    " (or __graft_entry__.build()); there is no CPU fallback"
                )
            L = ctypes.CDLL(str(LIB_PATH))
            _declare(L)
            _lib = L
    return _lib


def check(rc: int) -> None:
    if rc == RK_OK:
        return
    msg = lib().rk_last_error().decode("utf-8", "replace")
    if rc == RK_EINVAL:
        raise ValueError(msg)
    if rc == RK_ENCCL:
        raise RuntimeError(f"librkb200 (NCCL): {msg}")
    raise RuntimeError(f"librkb200: {msg}")


class Context:
    """One rk_ctx_t (per-device scratch: per-tile results, counter sets, pattern cache,
    staging rings); ``lock`` serialises the Python callers of a context."""

    def __init__(self, device: int):
        self.device = device
        h = ctypes.c_void_p()
        check(lib().rk_ctx_create(device, ctypes.byref(h)))
        self.handle = h
        self.lock = threading.Lock()

    def close(self) -> None:
        if self.handle:
            lib().rk_ctx_destroy(self.handle)
            self.handle = ctypes.c_void_p()

    @property
    def launches(self) -> int:
        return int(lib().rk_launch_count(self.handle))


_ctx: dict[int, Context] = {}
_ctx_lock = threading.Lock()


def default_device() -> int:
    env = os.environ.get("RKB200_DEVICE")
    if env is not None:
        return int(env)
    try:
        import torch

        if torch.cuda.is_available():
            return torch.cuda.current_device()
    except Exception:  # pragma: no cover - torch always present in this image
        pass
    return 0


def context(device: int | None = None) -> Context:
    if device is None:
        device = default_device()
    with _ctx_lock:
        c = _ctx.get(device)
        if c is None:
            c = Context(device)
            _ctx[device] = c
        return c


_spare: dict[int, list[Context]] = {}


class _Held:
    def __init__(self, ctx: Context, spare: bool):
        self.ctx, self.spare = ctx, spare

    def __enter__(self) -> Context:
        return self.ctx

    def __exit__(self, *exc) -> None:
        self.ctx.lock.release()
        if self.spare:
            with _ctx_lock:
                _spare.setdefault(self.ctx.device, []).append(self.ctx)


def acquire(device: int | None = None) -> _Held:
    """A context of ``device`` held for one call (``with acquire(dev) as ctx: ...``).

    The device's primary context when it is free, else a spare one from a per-device pool
    (created on demand): concurrent callers -- the reference runs range scans concurrently
    on a thread pool (parallel.py:111-121, :162-167) -- each get their own scratch and
    staging streams and run in parallel instead of queueing on one context."""
    if device is None:
        device = default_device()
    primary = context(device)
    if primary.lock.acquire(blocking=False):
        return _Held(primary, False)
    with _ctx_lock:
        pool = _spare.get(device)
        c = pool.pop() if pool else None
    if c is None:
        c = Context(device)
    c.lock.acquire()
    return _Held(c, True)


@atexit.register
def _close_all() -> None:  # pragma: no cover
    for c in list(_ctx.values()) + [x for v in _spare.values() for x in v]:
        try:
            c.close()
        except Exception:
            pass
    _ctx.clear()
    _spare.clear()


def u64ref(v: int = 0):
    return ctypes.c_uint64(v)
