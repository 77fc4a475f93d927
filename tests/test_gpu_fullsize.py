"""Bit-exactness at BASELINE.json's full sizes (configs[1..4]) against the CPU oracle.

Every test compares the B200 result with the oracle's EXACT result over the whole input
-- offsets, match count and collision count -- not with properties on a prefix.  The
oracle side regenerates each corpus on the host with its own restatement of the
reference generator (oracle.c_fill, datagen.py:68-77) and scans it with the reference's
per-window decisions carried by the reference's rolling update (oracle.c_scan_mt,
_scan.py:28-50 + rkhash.py:48-60) on every host core, so the device generator, the
shard map and the kernels are all checked independently at 1-16 GiB.

  C2  1 GiB printable ASCII, m = 4 ... 1024 (+ non-powers), sampled and generated
  C3  4 GiB printable ASCII, 1,024 patterns of m = 16 (and m = 32, 5, mixed at 1 GiB)
  C4  16 GiB DNA, m = 32, copies planted across every 2/4/8-way shard boundary; the
      2/4/8-way shard scans (halo, bias) are also run shard by shard on the one GPU
  C5  1 GiB of 'a', pattern 'aaaa' (8 GiB of offsets)
"""

import numpy as np
import pytest

import oracle
import paper_1810_01051_b200 as rk
from paper_1810_01051_b200 import _scan, datagen, sharded
from tests import _golden as G

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

GiB = 1 << 30


def _torch():
    import torch

    return torch


def _corpus(seed, n, alphabet):
    """(host ndarray from the oracle's generator, device tensor from rk_generate); the two
    are asserted byte-identical over the whole corpus."""
    torch = _torch()
    host = oracle.c_fill(seed, 0, n, alphabet)
    dev = rk.generate_tensor(rk.DnaSpec(seed, n, alphabet))
    step = 1 << 30
    for a in range(0, n, step):
        b = min(n, a + step)
        assert torch.equal(dev[a:b], torch.from_numpy(host[a:b]).to(dev.device)), a
    return host, dev


@pytest.fixture(scope="module")
def c2(gpu):
    return _corpus(42, GiB, G.ASCII)


def _plant_both(host, dev, pat, plants):
    """Copies pat at every offset on both sides; returns an undo list for the host."""
    torch = _torch()
    m = len(pat)
    p = torch.frombuffer(bytearray(pat), dtype=torch.uint8).to(dev.device)
    parr = np.frombuffer(pat, dtype=np.uint8)
    undo = []
    for x in plants:
        undo.append((x, host[x:x + m].copy()))
        host[x:x + m] = parr
        dev[x:x + m] = p
    return undo


def _undo(host, dev, undo):
    torch = _torch()
    for x, saved in reversed(undo):
        host[x:x + saved.size] = saved
        dev[x:x + saved.size] = torch.from_numpy(saved).to(dev.device)


C2_CASES = [(m, "sampled") for m in (4, 5, 7, 8, 12, 16, 20, 25, 32, 64, 65, 100, 128, 256, 512,
                                     800, 1024)] + [(m, "generated") for m in (4, 8, 16, 32)]


@pytest.mark.parametrize("m,source", C2_CASES)
def test_c2_1gib_exact(c2, m, source):
    host, dev = c2
    spec = rk.DnaSpec(42, GiB, G.ASCII)
    pat = datagen.make_pattern(dev, spec, m, source)
    # copies straddling 8 KiB tiles, 64 MiB staging chunks and the end of the text
    plants = [k * (1 << 14) - 7 for k in (1, 2, 1000)] + [(64 << 20) - m // 2, GiB - m]
    undo = _plant_both(host, dev, pat, plants)
    try:
        offs, k, coll, hits = _scan.scan_counts(dev, pat, rk.hash_full(pat), 0, GiB - m + 1)
        eo, ec = oracle.c_scan_mt(host, pat)
    finally:
        _undo(host, dev, undo)
    got = offs.cpu().numpy()
    assert k == eo.size and np.array_equal(got, eo), (m, source, k, eo.size)
    assert coll == ec, (m, source, coll, ec)
    assert hits == k + coll
    assert set(plants) <= set(got.tolist())


def test_c2_host_text_public_api(c2):
    """search_sequential on a pinned host copy of the 1 GiB corpus (rk_scan_host: chunked
    staging overlapped with the scan) equals the oracle, m = 8 and m = 4."""
    torch = _torch()
    host, dev = c2
    pinned = torch.from_numpy(host).pin_memory()
    for m in (4, 8):
        pat = datagen.make_pattern(dev, rk.DnaSpec(42, GiB, G.ASCII), m, "sampled")
        st = rk.ScanStats()
        r = rk.search_sequential(pinned.numpy(), pat, stats=st)
        eo, ec = oracle.c_scan_mt(host, pat)
        assert r.offsets == eo.tolist() and st.collisions == ec
        assert st.hash_hits == eo.size + ec and st.windows == GiB - m + 1


# ------------------------------------------------------------------------- C3
def _c3_patterns(host, n, P, m, seed=43, alphabet=G.ASCII):
    """bench_configs.c3: P/2 sampled at splitmix64 offsets, P/2 generated."""
    pats = []
    state = seed
    for _ in range(P // 2):
        draw, state = datagen.splitmix64(state)
        x = draw % (n - m + 1)
        pats.append(host[x:x + m].tobytes())
    for j in range(P - P // 2):
        pats.append(oracle.generate((seed ^ 0x5DEECE66D) + j, m, alphabet))
    return pats


def _oracle_multi(host, patterns):
    """search_multi (matcher.py:125-157) by length group on the host cores ->
    {deduped index: offsets}."""
    pats, by_length, _ = oracle.pattern_set(patterns)
    out = {}
    for m, members in by_length.items():
        if m > host.size:
            for i in members:
                out[i] = []
            continue
        for j, offs in oracle.c_search_multi_mt(host, [pats[i] for i in members]):
            out[members[j]] = offs.tolist()
    return out


@pytest.mark.parametrize("n,m", [(4 * GiB, 16), (GiB, 32), (GiB, 5), (GiB, 4)])
def test_c3_multi_exact(gpu, n, m):
    host, dev = _corpus(43, n, G.ASCII)
    pats = _c3_patterns(host, n, 1024, m)
    # a colliding pair ("ac"/"ba" at the tail) inside the set
    pats += [b"a" * (m - 2) + b"ac", b"a" * (m - 2) + b"ba"]
    got = rk.search_multi(dev, pats)
    exp = _oracle_multi(host, pats)
    assert len(got) == len(exp)
    total = 0
    for i, r in got:
        assert r.offsets == exp[i], (i, len(r.offsets), len(exp[i]))
        total += len(r.offsets)
    assert total >= 512  # every sampled pattern occurs at least once


def test_c3_mixed_lengths_exact(gpu):
    """C3's corpus with 1,024 patterns of 64 lengths (4..67) in one PatternSet."""
    n = GiB
    host, dev = _corpus(43, n, G.ASCII)
    pats = []
    state = 43
    for i in range(1024):
        m = 4 + i % 64
        draw, state = datagen.splitmix64(state)
        x = draw % (n - m + 1)
        pats.append(host[x:x + m].tobytes())
    got = rk.search_multi(dev, pats)
    exp = _oracle_multi(host, pats)
    for i, r in got:
        assert r.offsets == exp[i], i


# ------------------------------------------------------------------------- C4
C4_N = 16 * GiB


def _c4_plants(n, m):
    # a copy straddling every shard boundary of the 2-, 4- and 8-way strong partitions
    # (sharded.strong_shard), the 2^32 byte boundary and the end of the text
    cuts = set()
    for world in (2, 4, 8):
        for r in range(1, world):
            cuts.add(sharded.strong_shard(r, world, n, m)[0])
    # (neighbouring cuts of different world sizes are a few bytes apart: one copy
    # straddles all of them; copies never overlap, so each one stays a match)
    plants = []
    for x in sorted({c - m // 2 for c in cuts}) + [n - m]:
        if not plants or x >= plants[-1] + m:
            plants.append(x)
    for c in sorted(cuts) + [1 << 32]:
        assert any(x < c < x + m for x in plants), c
    return plants


@pytest.fixture(scope="module")
def c4(gpu):
    torch = _torch()
    spec = rk.DnaSpec(42, C4_N)
    dev = rk.generate_tensor(spec)
    m = 32
    pat = datagen.make_pattern(dev, spec, m, "sampled")
    plants = _c4_plants(C4_N, m)
    p = torch.frombuffer(bytearray(pat), dtype=torch.uint8).to(dev.device)
    for x in plants:
        dev[x:x + m] = p
    # the oracle regenerates the corpus piece by piece (never 16 GiB at once)
    eo, ec = oracle.c_scan_generated(42, C4_N, b"ACGT", pat, plants)
    yield dev, pat, plants, eo, ec
    del dev
    torch.cuda.empty_cache()


def test_c4_16gib_exact(c4):
    dev, pat, plants, eo, ec = c4
    m = len(pat)
    offs, k, coll, hits = _scan.scan_counts(dev, pat, rk.hash_full(pat), 0, C4_N - m + 1)
    got = offs.cpu().numpy()
    assert k == eo.size and np.array_equal(got, eo)
    assert coll == ec and hits == k + coll
    assert set(plants) <= set(got.tolist())
    assert got.max() > (1 << 32)


@pytest.mark.parametrize("world", [2, 4, 8])
def test_c4_16gib_shard_map(c4, world):
    """The strong 2/4/8-way partition run shard by shard on this GPU: each shard is a
    separate view of its bytes plus the (m-1)-byte halo, scanned from its own base and
    biased to global offsets; the rank-order concatenation equals the oracle, including
    the copies planted across every boundary, and the counters add up."""
    torch = _torch()
    dev, pat, plants, eo, ec = c4
    m = len(pat)
    hx = rk.hash_full(pat)
    parts, coll_total = [], 0
    for r in range(world):
        a, b, blo, bhi = sharded.strong_shard(r, world, C4_N, m)
        shard = dev[blo:bhi]
        offs, k, coll, hits = _scan.scan_counts(shard, pat, hx, a - blo, b - blo, out_bias=blo)
        parts.append(offs)
        coll_total += coll
    got = torch.cat(parts).cpu().numpy()
    assert np.array_equal(got, eo) and coll_total == ec


# ------------------------------------------------------------------------- C5
def test_c5_all_a_1gib(gpu):
    """1 GiB of 'a' with 'aaaa': every window matches (range(n - 3), collisions 0,
    tests/test_matcher.py:66-70); 8 GiB of ordered offsets."""
    torch = _torch()
    n = GiB
    t = torch.full((n,), 97, dtype=torch.uint8, device="cuda")
    offs, k, coll, hits = _scan.scan_counts(t, b"aaaa", rk.hash_full(b"aaaa"), 0, n - 3)
    assert k == n - 3 and coll == 0 and hits == n - 3
    assert torch.equal(offs, torch.arange(n - 3, device="cuda"))
    del offs
    # the same text through the bitmap output: every bit set
    bits, k2, c2_, h2 = _scan.scan_bitmap(t, b"aaaa", rk.hash_full(b"aaaa"), 0, n - 3,
                                          packed=True)
    assert (k2, c2_, h2) == (n - 3, 0, n - 3)
    full = (n - 3) // 32
    assert bool((bits[:full] == -1).all())


def test_c5_device_search_single_scan(gpu):
    """search_sequential on a CUDA tensor at C5 density issues exactly one scan: the
    offsets beyond the first buffer are re-emitted (rk_scan_fetch), never rescanned."""
    torch = _torch()
    from paper_1810_01051_b200 import _lib

    n = 1 << 28
    t = torch.full((n,), 97, dtype=torch.uint8, device="cuda")
    ctx = _lib.context(0)
    before = ctx.launches
    offs, k, coll, hits = _scan.scan_counts(t, b"aaaa", rk.hash_full(b"aaaa"), 0, n - 3)
    launches = ctx.launches - before
    assert k == n - 3 and torch.equal(offs, torch.arange(n - 3, device="cuda"))
    assert launches == 3  # scan + emit + the re-emit of the fetch
