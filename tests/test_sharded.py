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
