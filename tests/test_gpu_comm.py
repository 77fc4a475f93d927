"""The multi-GPU data plane behind the C ABI (rk_comm_init / rk_scan_sharded / rk_comm_fetch,
NCCL called from librkb200) on the one GPU of the test box: a single-rank communicator,
so every collective is real NCCL but no rank waits on another GPU.  The partition and the
rank-order merge across several ranks are covered by tests/test_sharded.py (gloo) and by
tests/test_gpu_fullsize.py::test_c4_16gib_shard_map (every shard's scan on this GPU)."""

import os
import socket

import numpy as np
import pytest

import oracle
import paper_1810_01051_b200 as rk
from paper_1810_01051_b200 import _scan, sharded

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def comm(gpu):
    c = sharded.Communicator(device=0)
    yield c
    c.close()


def test_comm_info(comm):
    info = comm.info()
    assert info["nranks"] == 1 and info["rank"] == 0 and info["nccl_version"] >= 21000


def test_sharded_scan_device_text(comm):
    import torch

    spec = rk.DnaSpec(42, 64 << 20)
    t = rk.generate_tensor(spec)
    pat = rk.datagen.make_pattern(t, spec, 12, "sampled")
    n, m = t.numel(), len(pat)
    offs, k, coll, hits = comm.scan(t, pat, 0, n - m + 1, 0)
    eo, ec = oracle.c_scan_mt(t.cpu().numpy(), pat)
    assert offs.cpu().numpy().tolist() == eo.tolist() and coll == ec and hits == k + coll
    # a window range inside a shard held from byte 1000 on (global offsets come back)
    a, b = 5000, (40 << 20)
    shard = t[1000: b + m - 1]
    offs2, k2, coll2, _ = comm.scan(shard, pat, a, b, 1000)
    sel = eo[(eo >= a) & (eo < b)]
    assert offs2.cpu().numpy().tolist() == sel.tolist()


def test_sharded_scan_host_text_and_fetch(comm):
    """A host shard is staged into HBM chunk by chunk; more matches than cap: the rest is
    fetched from the kept gather (no rescan)."""
    import torch

    n = 48 << 20
    host = np.full(n, 97, dtype=np.uint8)
    host[::1000] = 98
    offs, k, coll, hits = comm.scan(host, b"aaaa", 0, n - 3, 0, cap=1000)
    eo, ec = oracle.c_scan_mt(host, b"aaaa")
    assert k == eo.size and coll == ec == 0 and hits == k
    assert torch.equal(offs.cpu(), torch.from_numpy(eo))
    pinned = torch.from_numpy(host).pin_memory()
    offs, k, _, _ = comm.scan(pinned, b"aab", 0, n - 2, 0)
    assert offs.cpu().numpy().tolist() == oracle.c_scan_mt(host, b"aab")[0].tolist()


def test_sharded_dense_all_a(comm):
    """C5 density through the exact allgather-v: 256 MiB of 'a', every window matches."""
    import torch

    n = 1 << 28
    t = torch.full((n,), 97, dtype=torch.uint8, device="cuda")
    offs, k, coll, hits = comm.scan(t, b"aaaa", 0, n - 3, 0, cap=n)
    assert k == n - 3 and coll == 0
    assert torch.equal(offs, torch.arange(n - 3, device="cuda"))


def test_sharded_edge_cases(comm):
    import torch

    t = torch.frombuffer(bytearray(b"acXba" * 10), dtype=torch.uint8).cuda()
    offs, k, coll, hits = comm.scan(t, b"ac", 0, t.numel() - 1, 0)
    assert offs.cpu().tolist() == list(range(0, 50, 5)) and coll == 10 and hits == 20
    offs, k, coll, hits = comm.scan(t, b"ac", 3, 3, 0)  # this rank owns no windows
    assert k == coll == hits == 0
    with pytest.raises(ValueError):
        comm.scan(t[10:], b"ac", 0, 30, 10)  # windows before the held bytes
    with pytest.raises(ValueError):
        comm.scan(t, b"ac", 0, t.numel(), 0)  # last window runs past the held bytes


def test_search_matches_search_sequential(comm):
    text = rk.generate(rk.DnaSpec(7, 1 << 20))
    for pat in (text[100:108], text[5000:5040], b"ACGTACGTAC"):
        st = rk.ScanStats()
        r = comm.search(text, pat, len(text), stats=st)
        st2 = rk.ScanStats()
        assert r == rk.search_sequential(text, pat, stats=st2)
        assert (st.windows, st.hash_hits, st.collisions) == \
            (st2.windows, st2.hash_hits, st2.collisions)


def test_communicator_over_torch_distributed(gpu):
    """The unique id shipped through a torch.distributed group (NCCL backend, 1 rank)."""
    import torch.distributed as dist

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("nccl", rank=0, world_size=1)
    try:
        c = sharded.Communicator()
        text = rk.generate(rk.DnaSpec(3, 1 << 16))
        assert c.search(text, text[77:90], len(text)) == rk.search_naive(text, text[77:90])
        c.close()
    finally:
        dist.destroy_process_group()


def test_sharded_multi_pattern(comm):
    """rk_multi_scan_sharded (one rank): the pairs of a whole PatternSet -- short, q-gram
    and mixed lengths -- equal search_multi's, and a sub-range of starts held from
    byte 1000 on reports exactly its starts (global offsets)."""
    import torch

    rng = np.random.default_rng(44)
    n = 3 << 20
    host = rng.integers(0, 4, n, dtype=np.uint8) + 65
    pats = [host[x:x + m].tobytes() for x, m in ((10, 4), (5000, 6), (77777, 9), (2 << 20, 20),
                                                   (n - 33, 33))]
    pats += [b"ACGT", b"TTTTTTTTTTTTTT"]
    text = torch.from_numpy(host).cuda()
    got = comm.search_multi(text, pats, n)
    assert got == rk.search_multi(text, pats)
    # starts [5000, 2 MiB) held from byte 1000 (+ the 32-byte halo)
    a, b, blo = 5000, 2 << 20, 1000
    idx, off = comm.multi_scan(text[blo: b + 32], pats, a, b, blo, n)
    ps = rk.PatternSet(pats)
    full = dict(rk.search_multi(host.tobytes(), ps))
    for i in range(len(ps)):
        exp = [x for x in full[i].offsets if a <= x < b]
        assert off[idx == i].cpu().tolist() == exp, i


def test_sharded_batch(comm):
    """rk_scan_sharded_batch (one rank): nine patterns over one device shard in one
    collective equal rk_scan_sharded per pattern, including a dense pattern that overflows
    its first local buffer (second round) and an output cap below the total (not written,
    totals still returned)."""
    import torch

    rng = np.random.default_rng(45)
    n = 16 << 20
    host = rng.integers(0, 4, n, dtype=np.uint8) + 65
    host[(1 << 20): (1 << 20) + 200000] = 65  # an 'AAAA' run: a dense pattern
    t = torch.from_numpy(host).cuda()
    pats = [host[x:x + m].tobytes() for x, m in ((100, 4), (5000, 8), (70000, 16), (9 << 20, 32),
                                                   (123, 64), (4567, 128), (99, 256))]
    pats += [b"AAAA", b"ACGTACGTTT"]
    ranges = [(1000, n - len(p) + 1 - 7) for p in pats]
    outs = [torch.empty(1 << 20, dtype=torch.int64, device="cuda") for _ in pats]
    outs[-1] = torch.empty(1, dtype=torch.int64, device="cuda")  # too small for its list
    res = comm.scan_batch(t, pats, ranges, 0, outs)
    for p, (lo, hi), (offs, k, coll, hits) in zip(pats, ranges, res):
        e_offs, e_k, e_coll, e_hits = comm.scan(t, p, lo, hi, 0, cap=1 << 20)
        assert (k, coll, hits) == (e_k, e_coll, e_hits)
        if offs is not None:
            assert torch.equal(offs, e_offs)
    assert res[7][1] > 100000  # the dense one
    # the second call reuses the grown buffers (a steady workload pays the second round once)
    res2 = comm.scan_batch(t, pats, ranges, 0, outs)
    assert [r[1:] for r in res2] == [r[1:] for r in res]


def test_sharded_batch_async(comm):
    """rk_scan_sharded_batch_async (one rank): the same lists and totals as the synchronous
    batch, with no host round trip; a pattern over its slab reports overflow, an output
    cap below the total keeps only its prefix; back-to-back calls stay exact."""
    import torch

    rng = np.random.default_rng(46)
    n = 16 << 20
    host = rng.integers(0, 4, n, dtype=np.uint8) + 65
    host[(2 << 20): (2 << 20) + 50000] = 65
    t = torch.from_numpy(host).cuda()
    pats = [host[x:x + m].tobytes() for x, m in ((100, 4), (5000, 8), (70000, 16), (9 << 20, 32),
                                                   (123, 64), (4567, 128))]
    pats += [b"AAAA", b"ACGTACGTTT"]
    ranges = [(1000, n - len(p) + 1 - 7) for p in pats]
    ref_outs = [torch.empty(1 << 20, dtype=torch.int64, device="cuda") for _ in pats]
    ref = comm.scan_batch(t, pats, ranges, 0, ref_outs)
    outs = [torch.full((1 << 20,), -1, dtype=torch.int64, device="cuda") for _ in pats]
    outs[1] = torch.full((3,), -1, dtype=torch.int64, device="cuda")  # a cap below the total
    counts = torch.zeros((len(pats), 4), dtype=torch.int64, device="cuda")
    slab = 8192
    for _ in range(3):
        comm.scan_batch_async(t, pats, ranges, 0, outs, counts, slab=slab)
    torch.cuda.synchronize()
    c = counts.cpu().numpy()
    for i, (offs, k, coll, hits) in enumerate(ref):
        assert (int(c[i, 0]), int(c[i, 1]), int(c[i, 2])) == (k, hits, coll), i
        assert int(c[i, 3]) == (1 if k > slab else 0), i
        if k <= slab:
            w = min(k, outs[i].numel())
            assert torch.equal(outs[i][:w], offs[:w]), i
    assert int(c[6, 3]) == 1  # the 'AAAA' run is over the slab


def test_sharded_batch_async_edges(comm):
    """The asynchronous batch at its limits: 64 patterns (RK_BATCH_MAX_PATTERNS), some with
    no windows (win_hi <= win_lo) or no output (cap 0), a slab of one offset; every total
    equals the synchronous batch's and the overflow flags say which lists are complete."""
    import torch

    rng = np.random.default_rng(47)
    n = 4 << 20
    host = rng.integers(0, 4, n, dtype=np.uint8) + 65
    t = torch.from_numpy(host).cuda()
    pats = [host[x:x + m].tobytes() for x, m in zip(rng.integers(0, n - 64, 64), rng.integers(3, 40, 64))]
    ranges = [(100, n - len(p) + 1) if i % 7 else (500, 500) for i, p in enumerate(pats)]
    ref_outs = [torch.empty(1 << 16, dtype=torch.int64, device="cuda") for _ in pats]
    ref = comm.scan_batch(t, pats, ranges, 0, ref_outs)
    outs = [torch.full((1 << 16,) if i % 5 else (0,), -1, dtype=torch.int64, device="cuda")
            for i in range(len(pats))]
    counts = torch.zeros((len(pats), 4), dtype=torch.int64, device="cuda")
    comm.scan_batch_async(t, pats, ranges, 0, outs, counts, slab=1)
    torch.cuda.synchronize()
    c = counts.cpu().numpy()
    for i, (offs, k, coll, hits) in enumerate(ref):
        assert (int(c[i, 0]), int(c[i, 1]), int(c[i, 2])) == (k, hits, coll), i
        assert int(c[i, 3]) == (1 if k > 1 else 0), i
        if k == 1 and outs[i].numel():
            assert torch.equal(outs[i][:1], offs[:1]), i
        if i % 7 == 0:
            assert k == 0
