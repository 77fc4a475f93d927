"""Matcher core -- drop-in for rkmatch.matcher (/root/reference/pkg/src/rkmatch/matcher.py).

``MatchResult``, ``ScanStats``, ``PatternSet``, ``search_naive`` and
``search_sequential`` keep the reference's fields, signatures, validation order and
exceptions; ``search_multi`` returns the same ``[(index, MatchResult)]`` list.  The hash
sweeps run on the B200 (``_scan`` / ``rk_multi_scan``); ``search_naive`` stays the
brute-force definition the reference ships as its oracle.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _lib, _scan
from .rkhash import hash_full


@dataclass
class MatchResult:
    """All match offsets for one (text, pattern) search (matcher.py:23-42).

    Offsets are ascending, unique, in [0, text_length - pattern_length], and the window
    at every reported offset byte-equals the pattern."""

    text_length: int
    pattern_length: int
    offsets: list[int]

    def to_bitmap(self) -> np.ndarray:
        """Dense per-window boolean map, True where a match starts."""
        n_windows = max(self.text_length - self.pattern_length + 1, 0)
        bitmap = np.zeros(n_windows, dtype=bool)
        if self.offsets:
            bitmap[np.asarray(self.offsets)] = True
        return bitmap


@dataclass
class ScanStats:
    """Counters of an instrumented scan (matcher.py:45-55): hash_hits = matches + collisions."""

    windows: int = 0
    hash_hits: int = 0
    collisions: int = 0


class PatternSet:
    """Deduplicated non-empty patterns indexed for one-pass multi search (matcher.py:58-87)."""

    def __init__(self, patterns):
        self.patterns: list[bytes] = []
        self.by_length: dict[int, list[int]] = {}
        self.hash_index: dict[int, dict[int, list[int]]] = {}
        seen: set[bytes] = set()
        for raw in patterns:
            p = bytes(raw)
            if not p:
                raise ValueError("empty pattern")
            if p in seen:
                continue
            seen.add(p)
            idx = len(self.patterns)
            self.patterns.append(p)
            m = len(p)
            self.by_length.setdefault(m, []).append(idx)
            self.hash_index.setdefault(m, {}).setdefault(hash_full(p), []).append(idx)
        if not self.patterns:
            raise ValueError("pattern set is empty")

    def __len__(self) -> int:
        return len(self.patterns)


def _to_list(offsets) -> list[int]:
    return offsets.tolist()


def search_naive(text, pattern) -> MatchResult:
    """Ground-truth definition: direct byte comparison at every offset (matcher.py:90-98)."""
    text = text if isinstance(text, bytes) else bytes(text)
    pattern = pattern if isinstance(pattern, bytes) else bytes(pattern)
    if not pattern:
        raise ValueError("empty pattern")
    n, m = len(text), len(pattern)
    offsets = [x for x in range(n - m + 1) if text[x : x + m] == pattern]
    return MatchResult(n, m, offsets)


def search_sequential(text, pattern, stats: ScanStats | None = None) -> MatchResult:
    """Hash every window, byte-verify on hash equality (matcher.py:101-122), on the B200."""
    t = _scan.as_u8(text)
    p = _scan.as_u8(pattern)
    m = _scan._size(p)
    if m == 0:
        raise ValueError("empty pattern")
    n = _scan._size(t)
    n_windows = n - m + 1
    if n_windows <= 0:
        return MatchResult(n, m, [])
    hx = hash_full(p)
    offsets, matches, collisions, hash_hits = _scan.scan_counts(t, p, hx, 0, n_windows)
    if stats is not None:
        stats.windows += n_windows
        stats.hash_hits += hash_hits
        stats.collisions += collisions
    return MatchResult(n, m, _to_list(offsets))


def search_each(text, patterns, stats: ScanStats | None = None) -> list[MatchResult]:
    """``[search_sequential(text, p, stats) for p in patterns]`` -- the reference CLI's
    per-pattern loop over a pattern file (cli.py:105-118) -- with a host text crossing
    PCIe once for all of them (rk_scan_host_batch: the text lands chunk by chunk and every
    pattern's windows are scanned as their bytes arrive).  Patterns keep their order and
    duplicates (unlike search_multi's PatternSet); validation is search_sequential's, in
    the same order, before any device work; ``stats`` accumulates over all patterns."""
    t = _scan.as_u8(text)
    pats = [_scan._host_bytes(_scan.as_u8(p)) for p in patterns]
    for p in pats:
        if p.size == 0:
            raise ValueError("empty pattern")
    n = _scan._size(t)
    if _scan._device_of(t) is not None or not pats:
        return [search_sequential(t, p, stats) for p in pats]
    host = _scan._host_bytes(t)
    L = _lib.lib()
    out: list[MatchResult] = []
    for a in range(0, len(pats), _lib.BATCH_MAX_PATTERNS):
        batch = pats[a:a + _lib.BATCH_MAX_PATTERNS]
        P = len(batch)
        flat = np.concatenate(batch)
        lengths = np.array([p.size for p in batch], dtype=np.uint32)
        hashes = np.array([hash_full(p.tobytes()) for p in batch], dtype=np.uint64)
        mt = np.zeros(P, dtype=np.uint64)
        co = np.zeros(P, dtype=np.uint64)
        hh = np.zeros(P, dtype=np.uint64)
        cap = 1 << 16
        offs = np.empty(cap, dtype=np.int64)
        with _lib.acquire() as ctx:
            _lib.check(L.rk_scan_host_batch(ctx.handle, _scan._ptr(host), n, flat.ctypes.data,
                                            lengths.ctypes.data, hashes.ctypes.data, P,
                                            offs.ctypes.data, cap, mt.ctypes.data,
                                            co.ctypes.data, hh.ctypes.data))
            total = int(mt.sum())
            if total > cap:
                offs = np.empty(total, dtype=np.int64)
                _lib.check(L.rk_scan_host_fetch(ctx.handle, offs.ctypes.data, 0, total))
        at = 0
        for i, p in enumerate(batch):
            k = int(mt[i])
            m = int(p.size)
            nw = n - m + 1
            out.append(MatchResult(n, m, offs[at:at + k].tolist() if nw > 0 else []))
            at += k
            if stats is not None and nw > 0:
                stats.windows += nw
                stats.hash_hits += int(hh[i])
                stats.collisions += int(co[i])
    return out


def search_bitmap(text, pattern, stats: ScanStats | None = None):
    """search_sequential(text, pattern).to_bitmap() computed on the device without the
    offset list (matcher.py:36-42 + :101-122): a bool array/tensor with one entry per
    window, True where a match starts."""
    t = _scan.as_u8(text)
    p = _scan.as_u8(pattern)
    m = _scan._size(p)
    if m == 0:
        raise ValueError("empty pattern")
    n = _scan._size(t)
    n_windows = n - m + 1
    if n_windows <= 0:
        return np.zeros(0, dtype=bool)
    bits, matches, collisions, hash_hits = _scan.scan_bitmap(t, p, hash_full(p), 0, n_windows)
    if stats is not None:
        stats.windows += n_windows
        stats.hash_hits += hash_hits
        stats.collisions += collisions
    return bits


def _device_text(t):
    """(device tensor, device index) for search_multi; host text is copied once."""
    import torch

    if _scan._device_of(t) is not None:
        return t, _scan._device_of(t)
    dev = _lib.default_device()
    return _scan.to_device(_scan._host_bytes(t), dev), dev


def multi_scan(t_dev, dev: int, pats: list[bytes]):
    """Patterns of any lengths through rk_multi_scan_mixed (one device sweep for all lengths
    >= 7, one for 4..6, one for 1..3) -> [offsets ndarray per pattern]."""
    import torch

    L = _lib.lib()
    P = len(pats)
    n = int(t_dev.numel())
    flat = np.frombuffer(b"".join(pats), dtype=np.uint8)
    lengths = np.array([len(p) for p in pats], dtype=np.uint32)
    hashes = np.array([hash_full(p) for p in pats], dtype=np.uint64)
    stream = _scan._stream(dev)
    # pairs beyond cap are counted but not written (the sweep then runs again with exact
    # room): room for the text's own size covers every set short of adversarial density
    cap = max(1 << 16, min(n, 1 << 24))
    pairs = _lib.u64ref()
    for _attempt in range(2):
        off = torch.empty(cap, dtype=torch.int64, device=t_dev.device)
        idx = torch.empty(cap, dtype=torch.int32, device=t_dev.device)
        with _lib.acquire(dev) as ctx:
            _lib.check(L.rk_multi_scan_mixed(ctx.handle, t_dev.data_ptr(), n, flat.ctypes.data,
                                             lengths.ctypes.data, P, hashes.ctypes.data,
                                             off.data_ptr(), idx.data_ptr(), cap,
                                             ctypes.byref(pairs), stream))
        k = int(pairs.value)
        if k <= cap:
            break
        cap = k
    off = off[:k].cpu().numpy()
    idx = idx[:k].cpu().numpy()
    bounds = np.searchsorted(idx, np.arange(P + 1), side="left")
    return [off[bounds[i] : bounds[i + 1]] for i in range(P)]


def search_multi(text, patterns) -> list[tuple[int, MatchResult]]:
    """Every pattern of a PatternSet (matcher.py:125-157): all lengths >= 7 in one device
    sweep (per 64 lengths), 4..6 in one more, 1..3 in another.

    Returns one (pattern index, MatchResult) per distinct pattern, in index order; each
    result equals search_naive for that pattern."""
    if not isinstance(patterns, PatternSet):
        patterns = PatternSet(patterns)
    t = _scan.as_u8(text)
    n = _scan._size(t)
    found: dict[int, list[int]] = {i: [] for i in range(len(patterns))}
    idxs = [i for i, p in enumerate(patterns.patterns) if len(p) <= n]
    if idxs:
        t_dev, dev = _device_text(t)
        for a in range(0, len(idxs), _lib.MULTI_MAX_PATTERNS):
            batch = idxs[a : a + _lib.MULTI_MAX_PATTERNS]
            per = multi_scan(t_dev, dev, [patterns.patterns[i] for i in batch])
            for i, offs in zip(batch, per):
                found[i] = offs.tolist()
    return [
        (i, MatchResult(n, len(patterns.patterns[i]), found[i]))
        for i in range(len(patterns))
    ]
