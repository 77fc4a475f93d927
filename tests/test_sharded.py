"""Multi-rank host logic of the sharded scan (paper_1810_01051_b200/sharded.py) on CPU:
world_size 2 and 3 over gloo.  Each rank holds only its shard plus the (m-1)-byte halo;
the per-shard scan is the CPU oracle (test infrastructure standing in for the kernel),
so these tests check the partition, halo, gather order and counter reduction -- the
parts that run unchanged over NCCL on B200s."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_1810_01051_b200 import sharded


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _oracle_scan(shard, pattern, a, b):
    t = shard.numpy() if isinstance(shard, torch.Tensor) else shard
    p = np.frombuffer(pattern, dtype=np.uint8)
    offs, coll = oracle.c_scan(t, p, a, b)
    hits = len(offs) + coll
    return torch.from_numpy(offs.astype(np.int64)), len(offs), coll, hits


def _worker(rank, world, port, text, pattern, mode, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        n = len(text)
        m = len(pattern)
        if mode == "strong":
            a, b, blo, bhi = sharded.strong_shard(rank, world, n, m)
        else:
            per = -(-n // world)
            a, b, blo, bhi = sharded.weak_shard(rank, per, n, m)
        shard = torch.from_numpy(np.frombuffer(text, dtype=np.uint8)[blo:bhi].copy())
        offs, tot = sharded.search_sharded(shard, pattern, a, b, blo, scan_fn=_oracle_scan)
        q.put((rank, offs.tolist(), tot))
    finally:
        dist.destroy_process_group()


def _run(world, text, pattern, mode):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, text, pattern, mode, q))
             for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return sorted(out)


@pytest.mark.parametrize("world,mode", [(2, "strong"), (3, "weak"), (2, "weak")])
def test_sharded_gather_matches_oracle(world, mode):
    rng = np.random.default_rng(world * 7 + len(mode))
    n = 20000
    text = bytearray(rng.integers(0, 3, n, dtype=np.uint8).tobytes())
    pattern = bytes(text[100:117])
    # plant copies straddling every possible shard boundary
    for cut in (n // 2, n // 3, 2 * n // 3, -(-n // world), 2 * -(-n // world)):
        x = cut - 8
        if 0 <= x <= n - len(pattern):
            text[x : x + len(pattern)] = pattern
    text = bytes(text)
    expect, coll = oracle.c_scan(np.frombuffer(text, dtype=np.uint8),
                                 np.frombuffer(pattern, dtype=np.uint8))
    results = _run(world, text, pattern, mode)
    for rank, offs, tot in results:
        assert offs == expect.tolist()  # every rank holds the global ordered list
        assert tot == [len(expect), len(expect) + coll, coll]


def test_sharded_collisions_are_summed():
    text = b"ac" + b"Xba" * 3000
    results = _run(2, text, b"ac", "strong")
    for _, offs, tot in results:
        assert offs == [0]
        assert tot == [1, 3001, 3000]


def test_shard_maps_cover_windows_once():
    for n in (1, 5, 31, 1000, 4097):
        for m in (1, 3, 32):
            nw = max(n - m + 1, 0)
            for world in (1, 2, 3, 8):
                cov = []
                for r in range(world):
                    a, b, blo, bhi = sharded.strong_shard(r, world, n, m)
                    cov += list(range(a, b))
                    if b > a:
                        assert blo == a and bhi == b + m - 1 <= n
                assert cov == list(range(nw))
                per = -(-n // world)
                cov = []
                for r in range(world):
                    a, b, blo, bhi = sharded.weak_shard(r, per, n, m)
                    cov += list(range(a, b))
                assert cov == list(range(nw))


def _oracle_multi(shard, pats):
    t = shard.numpy() if isinstance(shard, torch.Tensor) else np.asarray(shard)
    ps, by_len, _ = oracle.pattern_set(pats)
    out = [None] * len(ps)
    for m, idxs in by_len.items():
        for j, offs in oracle.c_search_multi_group(t, [ps[i] for i in idxs]):
            out[idxs[j]] = offs
    return out


def _multi_worker(rank, world, port, text, pats, weak, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        n = len(text)
        lengths = [len(p) for p in pats]
        per = -(-n // world) if weak else None
        a, b, blo, bhi = sharded.multi_shard(rank, world, n, lengths, per)
        shard = torch.from_numpy(np.frombuffer(text, dtype=np.uint8)[blo:bhi].copy())
        idx, off = sharded.search_multi_sharded(shard, pats, a, b, blo, multi_fn=_oracle_multi)
        q.put((rank, idx.tolist(), off.tolist()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,weak", [(2, False), (3, True)])
def test_sharded_multi_pairs_match_oracle(world, weak):
    """Mixed lengths, copies straddling every shard boundary: each rank keeps the starts
    it owns (the (max m - 1)-byte halo serves the longest pattern), and the gathered
    pairs are the reference's per-pattern ascending lists."""
    rng = np.random.default_rng(40 + world)
    n = 12000
    text = bytearray(rng.integers(0, 3, n, dtype=np.uint8).tobytes())
    pats = [bytes(text[50 : 50 + m]) for m in (3, 9, 17, 40)] + [b"\x00\x01\x02" * 5]
    for cut in (n // 2, n // 3, 2 * n // 3, -(-n // world), 2 * -(-n // world)):
        for p in pats[1:4]:
            x = cut - len(p) // 2
            text[x : x + len(p)] = p
    text = bytes(text)
    expect = _oracle_multi(np.frombuffer(text, dtype=np.uint8), pats)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_multi_worker, args=(r, world, port, text, pats, weak, q))
             for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, idx, off in out:
        got = [[o for i, o in zip(idx, off) if i == j] for j in range(len(pats))]
        assert got == [e.tolist() for e in expect], rank


@pytest.mark.gpu
def test_sharded_multi_gpu_single_rank(gpu):
    """The default multi_fn (the B200 sweep) and the NCCL gather, one rank on cuda:0;
    the shard is a view into the middle of the text with its own start range."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(_free_port())
    dist.init_process_group("nccl", rank=0, world_size=1)
    try:
        rng = np.random.default_rng(9)
        n = 300000
        text = rng.integers(0, 4, n, dtype=np.uint8)
        pats = [text[x : x + m].tobytes() for x, m in ((10, 8), (5000, 20), (123456, 33))]
        a, b = 1000, 250000
        blo, bhi = a, min(b + 33 - 1, n)
        shard = torch.from_numpy(text[blo:bhi].copy()).cuda()
        idx, off = sharded.search_multi_sharded(shard, pats, a, b, blo)
        full = _oracle_multi(text, pats)
        for j in range(len(pats)):
            exp = [o for o in full[j].tolist() if a <= o < b]
            assert off[idx == j].cpu().tolist() == exp
    finally:
        dist.destroy_process_group()


def test_c_abi_shard_range_is_the_strong_partition():
    """rk_shard_range (C ABI, no GPU needed) == strong_shard (the partition of
    parallel.py:155-161) for every rank, including empty tails and m > n."""
    for n in (0, 1, 5, 31, 1000, 4097, 16 << 30):
        for m in (1, 3, 32, 1024):
            for world in (1, 2, 3, 4, 8):
                for r in range(world):
                    assert sharded.shard_range(n, m, world, r) == \
                        sharded.strong_shard(r, world, n, m), (n, m, world, r)


def _c4_worker(rank, world, port, seed, n, m, plants, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        a, b, blo, bhi = sharded.shard_range(n, m, world, rank)
        # the rank builds ONLY its bytes [blo, bhi): corpus slice + the planted copies
        # that intersect it (a copy straddling the cut lands half in each shard)
        buf = oracle.c_fill(seed, blo, bhi - blo, b"ACGT", threads=1)
        full_pat = plants["pattern"]
        for x in plants["at"]:
            lo, hi = max(x, blo), min(x + m, bhi)
            if lo < hi:
                buf[lo - blo: hi - blo] = np.frombuffer(full_pat[lo - x: hi - x], dtype=np.uint8)
        shard = torch.from_numpy(buf)
        offs, tot = sharded.search_sharded(shard, full_pat, a, b, blo, scan_fn=_oracle_scan)
        q.put((rank, offs.tolist(), tot))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_c4_shape_sharded_gloo(world):
    """BASELINE configs[3] at 4 MiB: DNA (seed 42), a sampled 32-byte pattern, copies
    planted across every 2/4/8-way shard cut; each rank regenerates only its shard + halo
    and the gathered list equals the oracle's scan of the whole text, on every rank."""
    n, m, seed = 4 << 20, 32, 42
    text = np.frombuffer(oracle.generate(seed, n), dtype=np.uint8)
    pat = oracle.make_pattern(text.tobytes(), seed, b"ACGT", m, "sampled")
    cuts = sorted({sharded.strong_shard(r, w, n, m)[0] for w in (2, 4, 8) for r in range(1, w)})
    at = []
    for x in [c - m // 2 for c in cuts]:
        if not at or x >= at[-1] + m:
            at.append(x)
    full = oracle.plant(text.tobytes(), pat, at)
    expect, coll = oracle.c_scan(np.frombuffer(full, dtype=np.uint8),
                                 np.frombuffer(pat, dtype=np.uint8))
    assert set(at) <= set(expect.tolist())
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_c4_worker,
                         args=(r, world, port, seed, n, m, {"pattern": pat, "at": at}, q))
             for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, offs, tot in out:
        assert offs == expect.tolist(), rank
        assert tot == [len(expect), len(expect) + coll, coll]
