"""CPU oracle for the reference scan path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its ``cpu_baseline``
leg and ``--impl reference``) may import this package, and only as the checker or as
the timed CPU baseline.  The product package ``paper_1810_01051_b200`` never imports
it; with its CUDA extension missing the product raises instead of falling back here.

Two layers restate the reference ``rkmatch`` package (/root/reference/pkg/src/rkmatch):

* pure Python / numpy restatements below (small cases, host semantics), each citing the
  reference file:line it follows;
* ``rk_oracle.c`` (built into ``oracle/build/librk_oracle.so`` by ``make -C oracle``),
  the same per-window algorithm in C for cases that must finish in seconds, and the
  multi-threaded ``search_parallel`` restatement used as the CPU baseline.

Parity is pinned: ``tests/test_oracle.py`` checks both layers against the golden
vectors in ``tests/golden/`` that ``tests/golden/make_golden.py`` produced by running
the reference itself.
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

import numpy as np

MASK64 = (1 << 64) - 1
_GOLDEN = 0x9E3779B97F4A7C15
_MIX1 = 0xBF58476D1CE4E5B9
_MIX2 = 0x94D049BB133111EB
_INITIAL_CAPACITY = 4096  # _scan.py:14
_HASH_BLOCK = 1 << 20  # matcher.py:20

_HERE = Path(__file__).resolve().parent
_LIB_PATH = _HERE / "build" / "librk_oracle.so"


# --------------------------------------------------------------------------- hashing
def hash_full(data) -> int:
    """rkhash.py:21-28: fold h = ((h << 1) + b) & MASK64; empty -> 0."""
    h = 0
    for b in bytes(data):
        h = ((h << 1) + b) & MASK64
    return h


def hash_window(text, offset: int, m: int) -> int:
    """rkhash.py:31-45."""
    if m < 1:
        raise ValueError("window length must be >= 1")
    if offset < 0 or offset + m > len(text):
        raise ValueError("window out of range")
    return hash_full(bytes(text[offset : offset + m]))


def roll(prev: int, outgoing: int, incoming: int, m: int) -> int:
    """rkhash.py:48-60."""
    if m < 1:
        raise ValueError("window length must be >= 1")
    top = (outgoing << (m - 1)) & MASK64
    return (((prev - top) << 1) + incoming) & MASK64


def window_hashes(text: np.ndarray, m: int, start: int, stop: int) -> np.ndarray:
    """_scan.py:71-91 (numpy, m passes of h <<= 1; h += text[...])."""
    if m < 1:
        raise ValueError("window length must be >= 1")
    if start == stop:
        return np.empty(0, dtype=np.uint64)
    if start < 0 or stop < start or stop - 1 + m > text.size:
        raise ValueError("window range out of bounds")
    count = stop - start
    h = np.zeros(count, dtype=np.uint64)
    for i in range(m):
        h <<= np.uint64(1)
        h += text[start + i : start + i + count]
    return h


# --------------------------------------------------------------------------- search
def as_u8(data) -> np.ndarray:
    """_scan.py:17-25."""
    if isinstance(data, np.ndarray):
        if data.dtype != np.uint8:
            raise TypeError(f"expected uint8 array, got {data.dtype}")
        return np.ascontiguousarray(data)
    if isinstance(data, (bytes, bytearray, memoryview)):
        return np.frombuffer(data, dtype=np.uint8)
    raise TypeError(f"expected bytes-like input, got {type(data).__name__}")


def search_naive(text, pattern) -> list[int]:
    """matcher.py:90-98: direct byte comparison at every offset (offsets only)."""
    text = bytes(text)
    pattern = bytes(pattern)
    if not pattern:
        raise ValueError("empty pattern")
    n, m = len(text), len(pattern)
    return [x for x in range(n - m + 1) if text[x : x + m] == pattern]


def scan_np(text: np.ndarray, pattern: np.ndarray, start: int, stop: int):
    """_scan.py:28-68 restated with numpy: hash every window of [start, stop), compare
    with hash_full(pattern), byte-verify the equal ones.  Returns (offsets int64[],
    collisions, hash_hits)."""
    m = pattern.size
    hx = np.uint64(hash_full(pattern.tobytes()))
    if stop <= start:
        return np.empty(0, np.int64), 0, 0
    offs = []
    coll = 0
    for a in range(start, stop, _HASH_BLOCK):
        b = min(a + _HASH_BLOCK, stop)
        h = window_hashes(text, m, a, b)
        cand = np.flatnonzero(h == hx) + a
        for x in cand.tolist():
            if np.array_equal(text[x : x + m], pattern):
                offs.append(x)
            else:
                coll += 1
    offs = np.asarray(offs, dtype=np.int64)
    return offs, coll, offs.size + coll


def search_sequential(text, pattern):
    """matcher.py:101-122 -> (n, m, offsets list, stats dict)."""
    t = as_u8(text)
    p = as_u8(pattern)
    if p.size == 0:
        raise ValueError("empty pattern")
    n, m = t.size, p.size
    nw = n - m + 1
    if nw <= 0:
        return n, m, [], {"windows": 0, "hash_hits": 0, "collisions": 0}
    offs, coll, hits = scan_np(t, p, 0, nw)
    return n, m, offs.tolist(), {"windows": nw, "hash_hits": hits, "collisions": coll}


def pattern_set(patterns):
    """matcher.py:66-84: dedupe (first occurrence), by_length, hash_index."""
    pats: list[bytes] = []
    seen: set[bytes] = set()
    by_length: dict[int, list[int]] = {}
    hash_index: dict[int, dict[int, list[int]]] = {}
    for raw in patterns:
        p = bytes(raw)
        if not p:
            raise ValueError("empty pattern")
        if p in seen:
            continue
        seen.add(p)
        idx = len(pats)
        pats.append(p)
        by_length.setdefault(len(p), []).append(idx)
        hash_index.setdefault(len(p), {}).setdefault(hash_full(p), []).append(idx)
    if not pats:
        raise ValueError("pattern set is empty")
    return pats, by_length, hash_index


def search_multi(text, patterns) -> list[tuple[int, list[int]]]:
    """matcher.py:125-157 -> [(idx, offsets)] in deduped index order."""
    pats, by_length, hash_index = pattern_set(patterns)
    t = as_u8(text)
    n = t.size
    found: dict[int, list[int]] = {i: [] for i in range(len(pats))}
    for m in sorted(by_length):
        nw = n - m + 1
        if nw <= 0:
            continue
        index = hash_index[m]
        for a in range(0, nw, _HASH_BLOCK):
            b = min(a + _HASH_BLOCK, nw)
            hashes = window_hashes(t, m, a, b)
            for hv, indices in index.items():
                for rel in np.flatnonzero(hashes == np.uint64(hv)):
                    x = a + int(rel)
                    w = t[x : x + m].tobytes()
                    for i in indices:
                        if w == pats[i]:
                            found[i].append(x)
    return [(i, sorted(found[i])) for i in range(len(pats))]


# --------------------------------------------------------------------------- launch algebra
def plan_launch(n: int, m: int, block_dim: int, axis_cap: int = 65535):
    """parallel.py:79-101 -> ((gx, gy, gz), block_dim)."""
    if not 1 <= block_dim <= 1024:
        raise ValueError("block_dim")
    if m < 1:
        raise ValueError("m")
    if m > n:
        raise ValueError("m > n")
    if axis_cap < 1:
        raise ValueError("axis cap")
    blocks = -(-(n - m + 1) // block_dim)
    gx, gy, gz = blocks, 1, 1
    if gx > axis_cap:
        gy = -(-gx // axis_cap)
        gx = axis_cap
        if gy > axis_cap:
            gz = -(-gy // axis_cap)
            gy = axis_cap
    return (gx, gy, gz), block_dim


# --------------------------------------------------------------------------- corpus
def splitmix64(state: int) -> tuple[int, int]:
    """datagen.py:28-34."""
    state = (state + _GOLDEN) & MASK64
    z = state
    z = ((z ^ (z >> 30)) * _MIX1) & MASK64
    z = ((z ^ (z >> 27)) * _MIX2) & MASK64
    return z ^ (z >> 31), state


def splitmix64_stream(seed: int, count: int, skip: int = 0) -> np.ndarray:
    """datagen.py:37-48 (vectorized counter form)."""
    steps = np.arange(skip + 1, skip + count + 1, dtype=np.uint64)
    z = np.uint64(seed & MASK64) + np.uint64(_GOLDEN) * steps
    z = (z ^ (z >> np.uint64(30))) * np.uint64(_MIX1)
    z = (z ^ (z >> np.uint64(27))) * np.uint64(_MIX2)
    return z ^ (z >> np.uint64(31))


def generate(seed: int, length: int, alphabet: bytes = b"ACGT") -> bytes:
    """datagen.py:68-77 via the C fill (bit-identical counter stream)."""
    lib = load()
    out = np.empty(length, dtype=np.uint8)
    if length:
        alpha = np.frombuffer(alphabet, dtype=np.uint8)
        lib.ro_splitmix64_fill(
            ctypes.c_uint64(seed & MASK64), ctypes.c_uint64(0), ctypes.c_uint64(length),
            alpha.ctypes.data, ctypes.c_uint32(len(alphabet)), out.ctypes.data,
        )
    return out.tobytes()


def plant(text, pattern, offsets) -> bytes:
    """datagen.py:80-102."""
    text = bytes(text)
    pattern = bytes(pattern)
    m = len(pattern)
    if m == 0:
        raise ValueError("empty pattern")
    ordered = sorted(offsets)
    for x in ordered:
        if x < 0 or x + m > len(text):
            raise ValueError("offset out of range")
    for a, b in zip(ordered, ordered[1:]):
        if b - a < m:
            raise ValueError("overlap")
    buf = bytearray(text)
    for x in ordered:
        buf[x : x + m] = pattern
    return bytes(buf)


def make_pattern(text: bytes, seed: int, alphabet: bytes, m: int, source: str) -> bytes:
    """bench.py:106-119 (_make_pattern)."""
    if source == "sampled":
        draw, _ = splitmix64(seed ^ 0xA5A5A5A5A5A5A5A5)
        x = draw % (len(text) - m + 1)
        return bytes(text[x : x + m])
    if source == "generated":
        return generate(seed ^ 0x5DEECE66D, m, alphabet)
    raise ValueError(source)


# --------------------------------------------------------------------------- C layer
_lib = None


def load():
    """Load oracle/build/librk_oracle.so (built by ``make -C oracle``)."""
    global _lib
    if _lib is not None:
        return _lib
    if not _LIB_PATH.exists():
        import subprocess

        subprocess.run(["make", "-s", "-C", str(_HERE)], check=True)
    lib = ctypes.CDLL(str(_LIB_PATH))
    u64, p = ctypes.c_uint64, ctypes.c_void_p
    lib.ro_hash_full.restype = u64
    lib.ro_hash_full.argtypes = [p, u64]
    lib.ro_scan_range.restype = u64
    lib.ro_scan_range.argtypes = [p, p, u64, u64, u64, u64, p, u64, ctypes.POINTER(u64)]
    lib.ro_scan_parallel.restype = u64
    lib.ro_scan_parallel.argtypes = [p, u64, p, u64, u64, u64, ctypes.c_int, p, u64,
                                     ctypes.POINTER(u64)]
    lib.ro_window_hashes.restype = None
    lib.ro_window_hashes.argtypes = [p, u64, u64, u64, p]
    lib.ro_search_multi.restype = u64
    lib.ro_search_multi.argtypes = [p, u64, p, p, ctypes.c_uint32, u64, p, p, u64, p]
    lib.ro_splitmix64_fill.restype = None
    lib.ro_splitmix64_fill.argtypes = [u64, u64, u64, p, ctypes.c_uint32, p]
    lib.ro_scan_roll_mt.restype = u64
    lib.ro_scan_roll_mt.argtypes = [p, p, u64, u64, u64, u64, ctypes.c_int, p, u64,
                                    ctypes.POINTER(u64)]
    lib.ro_fill_mt.restype = None
    lib.ro_fill_mt.argtypes = [u64, u64, u64, p, ctypes.c_uint32, p, ctypes.c_int]
    lib.ro_search_multi_mt.restype = u64
    lib.ro_search_multi_mt.argtypes = [p, u64, p, p, ctypes.c_uint32, u64, ctypes.c_int, p, p,
                                       u64, p]
    _lib = lib
    return lib


def c_scan(text: np.ndarray, pattern: np.ndarray, start: int = 0, stop: int | None = None,
           workers: int = 1):
    """C restatement of scan / search_parallel over windows [start, stop).

    workers == 1 runs _scan.py:53-68 on one range; workers > 1 runs the
    parallel.py:155-176 partition on pthreads (only for start == 0, full range).
    Returns (offsets int64[], collisions)."""
    lib = load()
    text = np.ascontiguousarray(text, dtype=np.uint8)
    pattern = np.ascontiguousarray(pattern, dtype=np.uint8)
    n, m = text.size, pattern.size
    nw = max(n - m + 1, 0)
    if stop is None:
        stop = nw
    hx = hash_full(pattern.tobytes())
    coll = ctypes.c_uint64(0)
    if workers == 1:
        cap = max(stop - start, 0)
        cap = min(cap, 1 << 16)
        out = np.empty(max(cap, 1), dtype=np.int64)
        k = lib.ro_scan_range(text.ctypes.data, pattern.ctypes.data, m, hx, start, stop,
                              out.ctypes.data, cap, ctypes.byref(coll))
        if k > cap:
            out = np.empty(k, dtype=np.int64)
            k = lib.ro_scan_range(text.ctypes.data, pattern.ctypes.data, m, hx, start, stop,
                                  out.ctypes.data, k, ctypes.byref(coll))
        return out[:k].copy(), int(coll.value)
    assert start == 0 and stop == nw
    cap = 1 << 16
    out = np.empty(cap, dtype=np.int64)
    k = lib.ro_scan_parallel(text.ctypes.data, n, pattern.ctypes.data, m, hx, nw, workers,
                             out.ctypes.data, cap, ctypes.byref(coll))
    if k > cap:
        out = np.empty(k, dtype=np.int64)
        k = lib.ro_scan_parallel(text.ctypes.data, n, pattern.ctypes.data, m, hx, nw, workers,
                                 out.ctypes.data, k, ctypes.byref(coll))
    return out[:k].copy(), int(coll.value)


def c_window_hashes(text: np.ndarray, m: int, start: int, stop: int) -> np.ndarray:
    lib = load()
    text = np.ascontiguousarray(text, dtype=np.uint8)
    out = np.empty(max(stop - start, 0), dtype=np.uint64)
    if out.size:
        lib.ro_window_hashes(text.ctypes.data, m, start, stop, out.ctypes.data)
    return out


def c_search_multi_group(text: np.ndarray, pats: list[bytes]):
    """C restatement of one equal-length group of search_multi.  Returns
    [(idx, offsets int64[])] in index order."""
    lib = load()
    text = np.ascontiguousarray(text, dtype=np.uint8)
    P = len(pats)
    m = len(pats[0])
    buf = np.frombuffer(b"".join(pats), dtype=np.uint8)
    ph = np.array([hash_full(p) for p in pats], dtype=np.uint64)
    counts = np.zeros(P, dtype=np.uint64)
    cap = 1 << 16
    offs = np.empty(cap, dtype=np.int64)
    idx = np.empty(cap, dtype=np.uint32)
    k = lib.ro_search_multi(text.ctypes.data, text.size, buf.ctypes.data, ph.ctypes.data, P, m,
                            offs.ctypes.data, idx.ctypes.data, cap, counts.ctypes.data)
    if k > cap:
        offs = np.empty(k, dtype=np.int64)
        idx = np.empty(k, dtype=np.uint32)
        k = lib.ro_search_multi(text.ctypes.data, text.size, buf.ctypes.data, ph.ctypes.data, P,
                                m, offs.ctypes.data, idx.ctypes.data, k, counts.ctypes.data)
    out = []
    base = 0
    for i in range(P):
        c = int(counts[i])
        out.append((i, offs[base : base + c].copy()))
        base += c
    return out


def cpu_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1


# --------------------------------------------------------------------------- full sizes
def c_scan_mt(text: np.ndarray, pattern, start: int = 0, stop: int | None = None,
              threads: int | None = None):
    """_scan.py:28-50 over windows [start, stop) with the reference's exact rolling update
    (rkhash.py:48-60) on pthreads: the checker for the 1-16 GiB configs.  `text` must hold
    the bytes [0, stop + m - 1).  Returns (offsets int64[], collisions)."""
    lib = load()
    text = np.ascontiguousarray(text, dtype=np.uint8)
    pat = np.frombuffer(bytes(pattern), dtype=np.uint8)
    m = pat.size
    if stop is None:
        stop = text.size - m + 1
    assert stop + m - 1 <= text.size
    threads = threads or cpu_threads()
    hx = hash_full(pat.tobytes())
    coll = ctypes.c_uint64(0)
    cap = 1 << 16
    out = np.empty(cap, dtype=np.int64)
    k = lib.ro_scan_roll_mt(text.ctypes.data, pat.ctypes.data, m, hx, start, stop, threads,
                            out.ctypes.data, cap, ctypes.byref(coll))
    if k > cap:
        out = np.empty(k, dtype=np.int64)
        k = lib.ro_scan_roll_mt(text.ctypes.data, pat.ctypes.data, m, hx, start, stop, threads,
                                out.ctypes.data, k, ctypes.byref(coll))
    return out[:k].copy(), int(coll.value)


def c_fill(seed: int, skip: int, count: int, alphabet: bytes = b"ACGT",
           threads: int | None = None) -> np.ndarray:
    """Bytes [skip, skip + count) of generate(seed, ..., alphabet) (datagen.py:68-77)."""
    lib = load()
    out = np.empty(count, dtype=np.uint8)
    if count:
        alpha = np.frombuffer(alphabet, dtype=np.uint8)
        lib.ro_fill_mt(ctypes.c_uint64(seed & MASK64), ctypes.c_uint64(skip),
                       ctypes.c_uint64(count), alpha.ctypes.data, ctypes.c_uint32(len(alphabet)),
                       out.ctypes.data, threads or cpu_threads())
    return out


def c_scan_generated(seed: int, n: int, alphabet: bytes, pattern, plants=(),
                     piece: int = 1 << 30, threads: int | None = None):
    """Scan the corpus generate(seed, n, alphabet) with `pattern` copied in at every
    offset of `plants` (datagen.py:80-102 semantics) WITHOUT materialising it: the corpus
    is regenerated on the host piece by piece (each piece carries the m - 1 bytes its last
    windows need) and scanned with c_scan_mt.  Returns (offsets int64[], collisions)."""
    pat = bytes(pattern)
    m = len(pat)
    parr = np.frombuffer(pat, dtype=np.uint8)
    nw = n - m + 1
    offs, coll = [], 0
    for a in range(0, nw, piece):
        b = min(a + piece, nw)
        buf = c_fill(seed, a, b - a + m - 1, alphabet, threads)
        for x in plants:
            lo, hi = max(x, a), min(x + m, a + buf.size)
            if lo < hi:
                buf[lo - a: hi - a] = parr[lo - x: hi - x]
        o, c = c_scan_mt(buf, pat, 0, b - a, threads)
        offs.append(o + a)
        coll += c
    return (np.concatenate(offs) if offs else np.empty(0, np.int64)), coll


def c_search_multi_mt(text: np.ndarray, pats: list[bytes], threads: int | None = None):
    """One equal-length group of search_multi (matcher.py:139-153) on pthreads.  Returns
    [(idx, offsets int64[])] in index order."""
    lib = load()
    text = np.ascontiguousarray(text, dtype=np.uint8)
    P = len(pats)
    m = len(pats[0])
    buf = np.frombuffer(b"".join(pats), dtype=np.uint8)
    ph = np.array([hash_full(p) for p in pats], dtype=np.uint64)
    counts = np.zeros(P, dtype=np.uint64)
    cap = 1 << 16
    offs = np.empty(cap, dtype=np.int64)
    idx = np.empty(cap, dtype=np.uint32)
    th = threads or cpu_threads()
    k = lib.ro_search_multi_mt(text.ctypes.data, text.size, buf.ctypes.data, ph.ctypes.data, P,
                               m, th, offs.ctypes.data, idx.ctypes.data, cap, counts.ctypes.data)
    if k > cap:
        offs = np.empty(k, dtype=np.int64)
        idx = np.empty(k, dtype=np.uint32)
        k = lib.ro_search_multi_mt(text.ctypes.data, text.size, buf.ctypes.data, ph.ctypes.data,
                                   P, m, th, offs.ctypes.data, idx.ctypes.data, k,
                                   counts.ctypes.data)
    out = []
    base = 0
    for i in range(P):
        c = int(counts[i])
        out.append((i, offs[base: base + c].copy()))
        base += c
    return out
