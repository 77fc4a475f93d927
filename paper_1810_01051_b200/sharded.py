"""Multi-GPU sharding: one process per GPU (torchrun), contiguous shards with halo.

The reference partitions the window range contiguously over workers and concatenates
the per-range lists in range order (/root/reference/pkg/src/rkmatch/parallel.py:155-172).
The same partition becomes the GPU shard map:

* rank r owns windows [a_r, b_r) and holds text bytes [a_r, b_r + m - 1) -- its shard
  plus an (m-1)-byte halo (the hash needs min(m,32)-1 of them, verification m-1);
* each rank scans its shard with no inter-GPU traffic;
* the only exchange is the final gather: per-rank counts, then every rank's positions
  over NVLink; concatenating in rank order is already the globally ascending list.

Two layers:

* ``Communicator`` -- the data plane behind the C ABI (rk_comm_init / rk_scan_sharded in
  librkb200.so, NCCL called from C++): each rank scans its shard (device tensor, or host
  memory staged chunk by chunk), then the counters are all-gathered and every rank's
  ordered positions are broadcast into every rank's output at its prefix -- an exact
  allgather-v, whatever the match density.  ``torch.distributed`` only ships the 128-byte
  NCCL unique id at setup.
* the ``torch.distributed`` helpers below (``search_sharded``, ``gather_offsets``, the
  multi-pattern gather), which take a process group, so the partition / halo / ordering
  logic is tested with ``gloo`` on CPU (tests/test_sharded.py).
"""

from __future__ import annotations

import ctypes

from . import _lib


def weak_shard(rank: int, per_rank: int, n_total: int, m: int) -> tuple[int, int, int, int]:
    """Weak scaling (fixed bytes per rank): rank r's windows start at r*per_rank.

    Returns (win_lo, win_hi, byte_lo, byte_hi) in global coordinates."""
    n_windows = max(n_total - m + 1, 0)
    a = min(rank * per_rank, n_windows)
    b = min((rank + 1) * per_rank, n_windows)
    return a, b, a, min(b + m - 1, n_total) if b > a else a


def strong_shard(rank: int, world: int, n_total: int, m: int) -> tuple[int, int, int, int]:
    """Strong scaling (fixed total): windows split as ceil(W/G) contiguous ranges."""
    n_windows = max(n_total - m + 1, 0)
    chunk = -(-n_windows // world) if n_windows else 0
    a = min(rank * chunk, n_windows)
    b = min(a + chunk, n_windows)
    return a, b, a, min(b + m - 1, n_total) if b > a else a


def gather_offsets(local, group=None):
    """All ranks' ascending offset lists concatenated in rank order (all_gather twice)."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    dev = local.device
    k = torch.tensor([local.numel()], dtype=torch.int64, device=dev)
    counts = [torch.zeros(1, dtype=torch.int64, device=dev) for _ in range(world)]
    dist.all_gather(counts, k, group=group)
    counts = [int(c) for c in torch.cat(counts).tolist()]  # one host round trip
    kmax = max(counts)
    if kmax == 0:
        return torch.empty(0, dtype=torch.int64, device=dev), counts
    padded = torch.zeros(kmax, dtype=torch.int64, device=dev)
    padded[: local.numel()] = local
    parts = [torch.empty(kmax, dtype=torch.int64, device=dev) for _ in range(world)]
    dist.all_gather(parts, padded, group=group)
    return torch.cat([p[:c] for p, c in zip(parts, counts)]), counts


def sum_counters(values, group=None):
    """All-reduce (sum) of per-rank integer counters (matches, hash_hits, collisions)."""
    import torch
    import torch.distributed as dist

    t = values if isinstance(values, torch.Tensor) else torch.tensor(values, dtype=torch.int64)
    dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return t


def search_sharded(shard, pattern, win_lo: int, win_hi: int, byte_lo: int, group=None,
                   scan_fn=None):
    """Scan this rank's shard (global windows [win_lo, win_hi), bytes from byte_lo) and
    gather the global ascending offsets on every rank.

    Returns (offsets tensor, [matches, hash_hits, collisions] summed over ranks).
    ``scan_fn(shard, pattern, start, stop) -> (offsets, matches, collisions, hash_hits)``
    defaults to the B200 scan."""
    import torch

    from . import _scan
    from .rkhash import hash_full

    if scan_fn is None:
        hx = hash_full(pattern)

        def scan_fn(t, p, a, b):
            return _scan.scan_counts(t, p, hx, a, b)

    if win_hi > win_lo:
        offs, k, coll, hits = scan_fn(shard, pattern, win_lo - byte_lo, win_hi - byte_lo)
        if not isinstance(offs, torch.Tensor):
            offs = torch.as_tensor(offs)
        offs = offs.to(torch.int64) + byte_lo
    else:
        dev = shard.device if isinstance(shard, torch.Tensor) else "cpu"
        offs, k, coll, hits = torch.empty(0, dtype=torch.int64, device=dev), 0, 0, 0
    allo, _ = gather_offsets(offs, group)
    tot = sum_counters(torch.tensor([k, hits, coll], dtype=torch.int64, device=offs.device), group)
    return allo, [int(v) for v in tot.tolist()]


def multi_shard(rank: int, world: int, n_total: int, lengths, per_rank: int | None = None):
    """Shard map of a multi-pattern search (matcher.py:125-157) over window STARTS: rank r
    owns starts [a_r, b_r) of the shortest length's start range and holds bytes
    [a_r, b_r + max(m) - 1) -- enough for the longest pattern starting in its range.
    ``per_rank`` given: weak scaling (fixed starts per rank), else strong."""
    m_min, m_max = min(lengths), max(lengths)
    if per_rank is None:
        a, b, _, _ = strong_shard(rank, world, n_total, m_min)
    else:
        a, b, _, _ = weak_shard(rank, per_rank, n_total, m_min)
    return a, b, a, min(b + m_max - 1, n_total) if b > a else a


def gather_pairs(idx, off, group=None):
    """All ranks' (pattern index, offset) pairs, ordered by (index, offset) on every rank.

    Each rank's pairs must already be in (index, offset) order and the ranks' start
    ranges ascending, so a stable sort by index of the rank-order concatenation is the
    global order (the reference's per-pattern ascending lists)."""
    import torch

    key = (idx.to(torch.int64) << 40) | off.to(torch.int64)  # offsets < 2^40
    allk, _ = gather_offsets(key, group)
    order = torch.sort(allk >> 40, stable=True).indices
    allk = allk[order]
    return (allk >> 40).to(torch.int32), allk & ((1 << 40) - 1)


def search_multi_sharded(shard, patterns, start_lo: int, start_hi: int, byte_lo: int,
                         group=None, multi_fn=None):
    """Multi-pattern search of this rank's shard (global starts [start_lo, start_hi),
    bytes from byte_lo), gathered on every rank.

    Returns (index int32 tensor, offset int64 tensor) ordered by (index, offset): pattern
    i's matches are the offsets of its run.  ``multi_fn(shard, patterns) -> [offsets per
    pattern]`` (shard-local) defaults to the B200 multi-pattern sweep."""
    import numpy as np
    import torch

    if multi_fn is None:
        from . import _scan
        from .matcher import _device_text, multi_scan

        def multi_fn(t, pats):
            t_dev, dev = _device_text(_scan.as_u8(t))
            return multi_scan(t_dev, dev, pats)

    from .matcher import PatternSet

    # pair indices are PatternSet indices (deduplicated, first occurrence), as search_multi's
    ps = patterns if isinstance(patterns, PatternSet) else PatternSet(patterns)
    dev = shard.device if isinstance(shard, torch.Tensor) else "cpu"
    idx_parts, off_parts = [], []
    if start_hi > start_lo:
        per = multi_fn(shard, list(ps.patterns))
        lo, hi = start_lo - byte_lo, start_hi - byte_lo
        for i, offs in enumerate(per):
            offs = torch.as_tensor(np.asarray(offs, dtype=np.int64))
            offs = offs[(offs >= lo) & (offs < hi)]  # halo starts belong to the next rank
            idx_parts.append(torch.full((offs.numel(),), i, dtype=torch.int32))
            off_parts.append(offs + byte_lo)
    idx = torch.cat(idx_parts) if idx_parts else torch.empty(0, dtype=torch.int32)
    off = torch.cat(off_parts) if off_parts else torch.empty(0, dtype=torch.int64)
    return gather_pairs(idx.to(dev), off.to(dev), group)


def shard_range(n_total: int, m: int, world: int, rank: int) -> tuple[int, int, int, int]:
    """rk_shard_range (the C ABI's strong partition, parallel.py:155-161): (win_lo, win_hi,
    byte_lo, byte_hi) of ``rank``; equal to strong_shard."""
    v = [_lib.u64ref() for _ in range(4)]
    _lib.check(_lib.lib().rk_shard_range(n_total, m, world, rank, *(ctypes.byref(x) for x in v)))
    return tuple(int(x.value) for x in v)


class Communicator:
    """This rank's NCCL communicator behind the C ABI (rk_comm_init).

    Collective: every rank of ``group`` (default: the default process group; none
    initialised = a single rank) constructs one.  Rank 0 draws the NCCL unique id
    (rk_comm_get_unique_id) and torch.distributed broadcasts those 128 bytes; nothing
    else goes through torch.distributed."""

    def __init__(self, group=None, device: int | None = None):
        import torch
        import torch.distributed as dist

        if dist.is_available() and dist.is_initialized():
            self.rank = dist.get_rank(group)
            self.world = dist.get_world_size(group)
        else:
            self.rank, self.world = 0, 1
        self.device = _lib.default_device() if device is None else device
        torch.cuda.set_device(self.device)
        L = _lib.lib()
        uid = (ctypes.c_uint8 * _lib.COMM_ID_BYTES)()
        if self.rank == 0:
            _lib.check(L.rk_comm_get_unique_id(uid))
        if self.world > 1:
            box = [bytes(uid) if self.rank == 0 else None]
            src = dist.get_global_rank(group, 0) if group is not None else 0
            dist.broadcast_object_list(box, src=src, group=group)
            uid = (ctypes.c_uint8 * _lib.COMM_ID_BYTES).from_buffer_copy(box[0])
        # a context of its own: the sharded scans' scratch never interleaves with other
        # callers' scans on the device's shared context
        self.ctx = _lib.Context(self.device)
        self._batch_key, self._batch_args = None, None
        h = ctypes.c_void_p()
        _lib.check(L.rk_comm_init(self.ctx.handle, uid, self.world, self.rank, ctypes.byref(h)))
        self.handle = h

    def close(self) -> None:
        if self.handle:
            _lib.lib().rk_comm_destroy(self.handle)
            self.handle = ctypes.c_void_p()
            self.ctx.close()

    def info(self) -> dict:
        n, r, v = ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
        _lib.check(_lib.lib().rk_comm_info(self.handle, ctypes.byref(n), ctypes.byref(r),
                                           ctypes.byref(v)))
        return {"nranks": n.value, "rank": r.value, "nccl_version": v.value}

    def scan(self, text, pattern, win_lo: int, win_hi: int, byte_lo: int, *,
             cap: int = 1 << 16, out=None, stream=None):
        """rk_scan_sharded: this rank's windows [win_lo, win_hi) of the global text, whose
        bytes [byte_lo, byte_lo + len(text)) it holds (CUDA tensor on this device, or host
        bytes / ndarray / pinned tensor).  Returns (global offsets as a CUDA int64 tensor,
        matches, collisions, hash_hits), totals over all ranks, on every rank."""
        import numpy as np
        import torch

        from . import _scan
        from .rkhash import hash_full

        L = _lib.lib()
        p = _scan._host_bytes(pattern)
        m = int(p.size)
        if m == 0:
            raise ValueError("empty pattern")
        t = _scan.as_u8(text)
        if isinstance(t, torch.Tensor) and not t.is_cuda:
            t = t.numpy()
        n = _scan._size(t)
        ptr = (t.data_ptr() if isinstance(t, torch.Tensor) else _scan._ptr(np.asarray(t))) if n else 0
        s = _scan._stream(self.device) if stream is None else stream
        if out is None:
            out = torch.empty(max(cap, 1), dtype=torch.int64, device=f"cuda:{self.device}")
        cap = min(cap, int(out.numel()))
        mt, co, hh = _lib.u64ref(), _lib.u64ref(), _lib.u64ref()
        with self.ctx.lock:
            _lib.check(L.rk_scan_sharded(self.handle, ptr, n, byte_lo, _scan._ptr(p), m,
                                         hash_full(p.tobytes()), win_lo, win_hi, out.data_ptr(),
                                         cap, ctypes.byref(mt), ctypes.byref(co),
                                         ctypes.byref(hh), s))
            k = int(mt.value)
            if k > cap:
                full = torch.empty(k, dtype=torch.int64, device=out.device)
                _lib.check(L.rk_comm_fetch(self.handle, full.data_ptr(), 0, k, s))
                out = full
        return out[:k], k, int(co.value), int(hh.value)

    def scan_batch(self, text, patterns, ranges, byte_lo: int, outs, stream=None):
        """rk_scan_sharded_batch: every pattern over its global windows ``ranges[i] =
        (win_lo, win_hi)`` of this rank's device shard (global bytes from byte_lo), the
        global ordered offsets into ``outs[i]`` (CUDA int64 tensors; written only when the
        list fits) -- one collective for all patterns.  Returns [(offsets view or None,
        matches, collisions, hash_hits)] per pattern, totals over all ranks."""
        import numpy as np

        from . import _scan

        L = _lib.lib()
        flat, lengths, hashes = self._batch_arrays(patterns)
        P = int(lengths.size)
        lo = np.array([r[0] for r in ranges], dtype=np.uint64)
        hi = np.array([r[1] for r in ranges], dtype=np.uint64)
        ptrs = np.array([o.data_ptr() for o in outs], dtype=np.uint64)
        caps = np.array([o.numel() for o in outs], dtype=np.uint64)
        mt, co, hh = (np.zeros(P, dtype=np.uint64) for _ in range(3))
        s = _scan._stream(self.device) if stream is None else stream
        with self.ctx.lock:
            _lib.check(L.rk_scan_sharded_batch(
                self.handle, text.data_ptr() if text.numel() else 0, int(text.numel()), byte_lo,
                flat.ctypes.data, lengths.ctypes.data, hashes.ctypes.data, P, lo.ctypes.data,
                hi.ctypes.data, ptrs.ctypes.data, caps.ctypes.data, mt.ctypes.data,
                co.ctypes.data, hh.ctypes.data, s))
        return [(outs[i][: int(mt[i])] if mt[i] <= caps[i] else None, int(mt[i]), int(co[i]),
                 int(hh[i])) for i in range(P)]

    def _batch_arrays(self, patterns):
        """(flat bytes, lengths, hashes) of a pattern list, kept for the next call with the
        same patterns (hash_full of a 1 KiB pattern in Python costs ~0.1 ms)."""
        import numpy as np

        from . import _scan
        from .rkhash import hash_full

        key = tuple(bytes(p) if isinstance(p, (bytes, bytearray, memoryview)) else None
                    for p in patterns)
        if None not in key and key == self._batch_key:
            return self._batch_args
        pats = [_scan._host_bytes(_scan.as_u8(p)) for p in patterns]
        args = (np.concatenate(pats), np.array([p.size for p in pats], dtype=np.uint32),
                np.array([hash_full(p.tobytes()) for p in pats], dtype=np.uint64))
        if None not in key:
            self._batch_key, self._batch_args = key, args
        return args

    def scan_batch_async(self, text, patterns, ranges, byte_lo: int, outs, counts, *,
                         slab: int = 4096, stream=None) -> None:
        """rk_scan_sharded_batch_async: as scan_batch, with no host round trip -- every
        rank's first ``slab`` ordered offsets per pattern are all-gathered in one NCCL
        group and ordered into ``outs[i]`` on the device; row i of ``counts`` (a CUDA int64
        tensor of P x 4) receives [matches, hash_hits, collisions, overflow], the totals
        over all ranks, stream-ordered; overflow = 1 when some rank found more than
        ``slab`` (the list is then incomplete: use scan_batch)."""
        import numpy as np

        from . import _scan

        L = _lib.lib()
        flat, lengths, hashes = self._batch_arrays(patterns)
        P = int(lengths.size)
        if counts.numel() < 4 * P or not counts.is_cuda:
            raise ValueError("counts must be a CUDA tensor of at least 4 x P int64")
        lo = np.array([r[0] for r in ranges], dtype=np.uint64)
        hi = np.array([r[1] for r in ranges], dtype=np.uint64)
        ptrs = np.array([o.data_ptr() for o in outs], dtype=np.uint64)
        caps = np.array([o.numel() for o in outs], dtype=np.uint64)
        s = _scan._stream(self.device) if stream is None else stream
        with self.ctx.lock:
            _lib.check(L.rk_scan_sharded_batch_async(
                self.handle, text.data_ptr() if text.numel() else 0, int(text.numel()), byte_lo,
                flat.ctypes.data, lengths.ctypes.data, hashes.ctypes.data, P, lo.ctypes.data,
                hi.ctypes.data, ptrs.ctypes.data, caps.ctypes.data, int(slab),
                counts.data_ptr(), s))

    def multi_scan(self, text, patterns, start_lo: int, start_hi: int, byte_lo: int,
                   n_total: int, *, cap: int = 1 << 16, stream=None):
        """rk_multi_scan_sharded: this rank's window starts [start_lo, start_hi) of the
        global text, whose bytes [byte_lo, byte_lo + len(text)) it holds on this device,
        against the PatternSet ``patterns``.  Returns every rank's pairs as (index int32
        tensor, offset int64 tensor) ordered by (index, offset), on every rank."""
        import numpy as np
        import torch

        from . import _scan
        from .matcher import PatternSet
        from .rkhash import hash_full

        L = _lib.lib()
        ps = patterns if isinstance(patterns, PatternSet) else PatternSet(patterns)
        flat = np.frombuffer(b"".join(ps.patterns), dtype=np.uint8)
        lengths = np.array([len(p) for p in ps.patterns], dtype=np.uint32)
        hashes = np.array([hash_full(p) for p in ps.patterns], dtype=np.uint64)
        t = _scan.as_u8(text)
        if not (isinstance(t, torch.Tensor) and t.is_cuda):
            t = _scan.to_device(_scan._host_bytes(t), self.device)
        n = int(t.numel())
        s = _scan._stream(self.device) if stream is None else stream
        pairs = _lib.u64ref()
        for _attempt in range(2):
            off = torch.empty(max(cap, 1), dtype=torch.int64, device=f"cuda:{self.device}")
            idx = torch.empty(max(cap, 1), dtype=torch.int32, device=f"cuda:{self.device}")
            with self.ctx.lock:
                _lib.check(L.rk_multi_scan_sharded(
                    self.handle, t.data_ptr() if n else 0, n, byte_lo, n_total, flat.ctypes.data,
                    lengths.ctypes.data, len(ps), hashes.ctypes.data, start_lo, start_hi,
                    off.data_ptr(), idx.data_ptr(), cap, ctypes.byref(pairs), s))
            k = int(pairs.value)
            if k <= cap:
                break
            cap = k
        return idx[:k], off[:k]

    def search_multi(self, shard, patterns, n_total: int):
        """search_multi's result over a text sharded across the ranks (multi_shard: each
        rank owns a contiguous range of window starts and holds the longest pattern's
        halo): ``shard`` is this rank's bytes, or the whole text (then sliced).  Returns
        [(pattern index, MatchResult)] of the whole text on every rank."""
        from . import _scan
        from .matcher import MatchResult, PatternSet

        ps = patterns if isinstance(patterns, PatternSet) else PatternSet(patterns)
        lengths = [len(p) for p in ps.patterns]
        fits = [m <= n_total for m in lengths]
        found = {i: [] for i in range(len(ps))}
        if any(fits):
            a, b, blo, bhi = multi_shard(self.rank, self.world, n_total,
                                         [m for m, f in zip(lengths, fits) if f])
            t = _scan.as_u8(shard)
            if _scan._size(t) == n_total and (blo, bhi) != (0, n_total):
                t = t[blo:bhi]
            idx, off = self.multi_scan(t, ps, a, b, blo, n_total)
            idx, off = idx.cpu().numpy(), off.cpu().numpy()
            import numpy as np

            bounds = np.searchsorted(idx, np.arange(len(ps) + 1), side="left")
            for i in range(len(ps)):
                found[i] = off[bounds[i]:bounds[i + 1]].tolist()
        return [(i, MatchResult(n_total, lengths[i], found[i])) for i in range(len(ps))]

    def search(self, shard, pattern, n_total: int, stats=None):
        """search_parallel's result over a text sharded across the ranks (strong partition,
        rk_shard_range): ``shard`` is this rank's bytes [byte_lo, byte_hi) -- or the whole
        text, which is then sliced.  Returns the global MatchResult on every rank."""
        from . import _scan
        from .matcher import MatchResult

        p = _scan._host_bytes(pattern)
        m = int(p.size)
        if m == 0:
            raise ValueError("empty pattern")
        if m > n_total:
            return MatchResult(n_total, m, [])
        a, b, blo, bhi = shard_range(n_total, m, self.world, self.rank)
        t = _scan.as_u8(shard)
        if _scan._size(t) == n_total and (blo, bhi) != (0, n_total):
            t = t[blo:bhi]
        offs, k, coll, hits = self.scan(t, p, a, b, blo)
        if stats is not None:
            stats.windows += n_total - m + 1
            stats.hash_hits += hits
            stats.collisions += coll
        return MatchResult(n_total, m, offs.cpu().tolist())
