"""GPU parity: the sm_100a scan against the golden vectors (produced by the reference)
and against the CPU oracle on seeded inputs.  Integer work: every comparison is
bit-exact (offsets, windows, hash_hits, collisions)."""

import hashlib

import numpy as np
import pytest

import oracle
import paper_1810_01051_b200 as rk
from paper_1810_01051_b200 import _scan
from tests import _golden as G

pytestmark = pytest.mark.gpu


def _torch():
    import torch

    return torch


def check_case(c, text_obj):
    st = rk.ScanStats()
    r = rk.search_sequential(text_obj, c["pattern"], stats=st)
    assert r.offsets == c["offsets"], c["tag"]
    assert (r.text_length, r.pattern_length) == (c["n"], c["m"])
    if c["m"] <= c["n"]:
        assert st.windows == c["windows"], c["tag"]
        assert st.hash_hits == c["hash_hits"], c["tag"]
        assert st.collisions == c["collisions"], c["tag"]


def test_golden_scan_cases_host_bytes(gpu):
    for c in G.scan_cases():
        check_case(c, c["text"])


def test_golden_scan_cases_device_tensors(gpu):
    torch = _torch()
    for c in G.scan_cases():
        t = torch.frombuffer(bytearray(c["text"]), dtype=torch.uint8).cuda() if c["n"] else \
            torch.empty(0, dtype=torch.uint8, device="cuda")
        check_case(c, t)


def test_golden_parallel_and_cfg_independence(gpu):
    for i, c in enumerate(G.scan_cases()):
        if i % 5 or c["m"] > c["n"]:
            continue
        for block in (1, 32, 1024):
            cfg = rk.plan_launch(c["n"], c["m"], block)
            st = rk.ScanStats()
            r = rk.search_parallel(c["text"], c["pattern"], cfg, workers=4, stats=st)
            assert r.offsets == c["offsets"] and st.collisions == c["collisions"], c["tag"]
        padded = rk.LaunchConfig((1024, 2, 2), 512)
        assert rk.search_parallel(c["text"], c["pattern"], padded, 3).offsets == c["offsets"]


def test_unaligned_device_views(gpu):
    """Text pointers at every offset mod 32 (the kernel's 256-bit loads are aligned down)."""
    torch = _torch()
    rng = np.random.default_rng(3)
    base = rng.integers(0, 4, 70000, dtype=np.uint8)
    base[rng.integers(0, 69000, 400)] = 7
    dev = torch.from_numpy(base).cuda()
    for shift in range(33):
        for m in (1, 3, 8, 17, 31, 32, 33, 40, 64, 70):
            n = 69000 - shift
            view = dev[shift : shift + n]
            host = base[shift : shift + n]
            pat = host[1234 : 1234 + m].tobytes()
            eo, ec = oracle.c_scan(host, np.frombuffer(pat, dtype=np.uint8), workers=4)
            st = rk.ScanStats()
            r = rk.search_sequential(view, pat, stats=st)
            assert r.offsets == eo.tolist(), (shift, m)
            assert st.collisions == ec, (shift, m)


def test_window_ranges_via_scan(gpu):
    """_scan.scan(text, pattern, hx, start, stop) on arbitrary sub-ranges."""
    torch = _torch()
    rng = np.random.default_rng(11)
    host = rng.integers(0, 3, 200000, dtype=np.uint8)
    dev = torch.from_numpy(host).cuda()
    for m in (2, 5, 12, 24, 29, 32, 48, 100):
        pat = host[777 : 777 + m]
        hx = oracle.hash_full(pat.tobytes())
        nw = host.size - m + 1
        for start, stop in [(0, nw), (1, 2), (5, 5), (16383, 16385), (12345, 170001),
                            (nw - 1, nw), (0, 1), (100, 33000)]:
            eo, ec = oracle.c_scan(host, pat, start, stop)
            do, dc = _scan.scan(dev, pat.tobytes(), hx, start, stop)
            assert do.cpu().numpy().tolist() == eo.tolist(), (m, start, stop)
            assert dc == ec
            ho, hc = _scan.scan(host, pat.tobytes(), hx, start, stop)
            assert ho.tolist() == eo.tolist() and hc == ec


def test_foreign_hx_semantics(gpu):
    """hx is a parameter (as in _scan_range): windows are hash-checked against it, then
    byte-verified against the pattern bytes."""
    rng = np.random.default_rng(5)
    host = rng.integers(97, 100, 60000, dtype=np.uint8)  # edge and staged (interior) tiles
    for m, hx_kind in [(1, "other"), (1, "big"), (2, "other"), (4, "other"), (5, "other"),
                       (6, "other"), (8, "other"), (12, "other"), (16, "other"), (20, "other"),
                       (30, "other"), (40, "other"), (70, "other")]:
        pat = host[100 : 100 + m]
        other = host[200 : 200 + m] if m > 1 else np.array([98], dtype=np.uint8)
        hx = oracle.hash_full(other.tobytes()) if hx_kind == "other" else 1000
        lib = oracle.load()
        import ctypes

        coll = ctypes.c_uint64()
        out = np.empty(host.size, dtype=np.int64)
        k = lib.ro_scan_range(host.ctypes.data, pat.ctypes.data, m, hx, 0, host.size - m + 1,
                              out.ctypes.data, out.size, ctypes.byref(coll))
        do, dc = _scan.scan(host, pat.tobytes(), hx, 0, host.size - m + 1)
        assert do.tolist() == out[:k].tolist() and dc == coll.value, m
    # unreachable hash for short windows
    do, dc = _scan.scan(b"abcabc", b"abc", 1 << 40, 0, 4)
    assert do.tolist() == [] and dc == 0


def test_random_fuzz_against_oracle(gpu):
    rng = np.random.default_rng(20240810)
    for case in range(600):
        k = (2, 3, 4, 256)[case % 4]
        n = int(rng.integers(1, 40000))
        m = int(rng.integers(1, 130))
        text = rng.integers(0, k, n, dtype=np.uint8)
        if m <= n and rng.random() < 0.6:
            x = int(rng.integers(0, n - m + 1))
            pat = text[x : x + m].copy()
        else:
            pat = rng.integers(0, k, m, dtype=np.uint8)
        st = rk.ScanStats()
        r = rk.search_sequential(text.tobytes(), pat.tobytes(), stats=st)
        if m > n:
            assert r.offsets == []
            continue
        eo, ec = oracle.c_scan(text, pat, workers=4)
        assert r.offsets == eo.tolist(), (case, n, m, k)
        assert st.collisions == ec, (case, n, m, k)
        assert st.hash_hits == len(eo) + ec


def test_short_patterns_density_mix(gpu):
    """m = 2..9 over texts whose hit density changes from tile to tile: sparse chunks go
    through the lane-flag pass + cooperative settle, dense ones through the inline settle
    (and the kernel's dense mode must switch back), at interior (staged) and edge tiles."""
    torch = _torch()
    rng = np.random.default_rng(5150)
    segs = []
    for i in range(24):
        kind = i % 4
        ln = int(rng.integers(3000, 40000))
        if kind == 0:
            segs.append(np.full(ln, ord("a"), dtype=np.uint8))
        elif kind == 1:
            segs.append(rng.integers(0, 2, ln, dtype=np.uint8) + ord("a"))
        elif kind == 2:
            segs.append(rng.integers(32, 127, ln, dtype=np.uint8))
        else:
            segs.append(rng.integers(0, 256, ln, dtype=np.uint8))
    text = np.concatenate(segs)
    dev = torch.from_numpy(text).cuda()
    for m in range(2, 10):
        for pat in (b"a" * m, bytes(text[50000 : 50000 + m]), bytes(rng.integers(32, 127, m, dtype=np.uint8))):
            eo, ec = oracle.c_scan(text, np.frombuffer(pat, dtype=np.uint8), workers=8)
            for off in (0, 5):
                st = rk.ScanStats()
                r = rk.search_sequential(dev[off:], pat, stats=st)
                want = [x - off for x in eo.tolist() if x >= off]
                assert r.offsets == want, (m, pat[:4], off)
                if off == 0:
                    assert st.collisions == ec and st.hash_hits == len(eo) + ec, (m, pat[:4])


def test_c1_sweep_golden(gpu):
    co = G.corpus()
    text = rk.generate(rk.DnaSpec(42, 2**20, G.ASCII))
    assert hashlib.sha256(text).hexdigest() == co["ascii_seed42_1MiB_sha256"]
    for e in co["ascii_seed42_1MiB_sweep"]:
        st = rk.ScanStats()
        r = rk.search_sequential(text, G.dec(e["pattern"]), stats=st)
        assert r.offsets == e["offsets"], (e["m"], e["source"])
        assert st.collisions == e["collisions"] and st.hash_hits == e["hash_hits"]
        assert st.windows == e["windows"]


def test_dna_planted_golden(gpu):
    co = G.corpus()
    dna = rk.generate(rk.DnaSpec(42, 4 * 2**20))
    assert hashlib.sha256(dna).hexdigest() == co["dna_seed42_4MiB_sha256"]
    assert hashlib.sha256(rk.generate(rk.DnaSpec(42, 2 * 2**20))).hexdigest() == \
        co["dna_seed42_2MiB_sha256"]
    for e in co["dna_seed42_4MiB"]:
        pat = G.dec(e["pattern"])
        text = rk.plant(dna, pat, e["plant"])
        st = rk.ScanStats()
        r = rk.search_sequential(text, pat, stats=st)
        assert r.offsets == e["offsets"] and st.collisions == e["collisions"]


def test_window_hashes_golden(gpu):
    torch = _torch()
    for e in G.hash_kat()["window_hashes"]:
        text = G.dec(e["text"])
        m = e["m"]
        h = _scan.window_hashes(np.frombuffer(text, dtype=np.uint8), m, 0, len(text) - m + 1)
        assert [int(v) for v in h.tolist()] == [int(v) for v in e["h"]]
        d = _scan.window_hashes(torch.frombuffer(bytearray(text), dtype=torch.uint8).cuda(), m, 1,
                                len(text) - m + 1)
        assert [int(v) for v in d.cpu().numpy().tolist()] == [int(v) for v in e["h"][1:]]
    with pytest.raises(ValueError):
        _scan.window_hashes(np.zeros(6, np.uint8), 3, 0, 5)
    with pytest.raises(ValueError):
        _scan.window_hashes(np.zeros(6, np.uint8), 0, 0, 1)


def test_generate_matches_oracle_slices(gpu):
    for seed, alpha in [(42, b"ACGT"), (43, G.ASCII), (7, b"ab"), (2**64 - 1, bytes(range(256)))]:
        spec = rk.DnaSpec(seed, 3 * 2**20 + 5, alpha)
        got = rk.generate(spec)
        assert got == oracle.generate(seed, spec.length, alpha)
        t = rk.generate_tensor(spec, skip=1000003, count=4099)
        assert t.cpu().numpy().tobytes() == got[1000003 : 1000003 + 4099]


def test_golden_multi_cases(gpu):
    for c in G.multi_cases():
        out = rk.search_multi(c["text"], rk.PatternSet(c["patterns"]))
        assert [[i, r.offsets] for i, r in out] == c["results"], c["tag"]
        for i, r in out:
            assert r.pattern_length == len(c["deduped"][i])


def test_multi_short_lengths_at_chunk_and_tile_edges(gpu):
    """m = 4..6 multi-pattern sets (anchored q-grams every 2 bytes + cuckoo lookups):
    occurrences planted so that windows end at every offset around 1 KiB chunk ends
    (their last bytes are the next chunk's), 4 KiB stage ends and 8 KiB tile ends, at the
    text's first and last bytes, and at unaligned device views."""
    torch = _torch()
    rng = np.random.default_rng(99)
    n = (1 << 20) + 37
    text = rng.integers(32, 127, n, dtype=np.uint8)
    for m in (4, 5, 6):
        pats = [rng.integers(32, 127, m, dtype=np.uint8).tobytes() for _ in range(40)]
        pats += [text[x : x + m].tobytes() for x in (0, n - m, 12345)]
        t = text.copy()
        # one intact occurrence per 1 KiB chunk end, ending d in [-3, 2] bytes from it
        # (cycling), so every stage end (4 KiB) and tile end (8 KiB) gets each d
        for k, base in enumerate(range(1024, n - 64, 1024)):
            d = (k // 8) % 6 - 3
            y = base + d - m + 1
            t[y : y + m] = np.frombuffer(pats[k % len(pats)], dtype=np.uint8)
        want = oracle.search_multi(t.tobytes(), pats)
        dev = torch.from_numpy(t).cuda()
        for off in (0, 3):
            got = rk.search_multi(dev[off:], pats)
            exp = [(i, [x - off for x in offs if x >= off]) for i, offs in want]
            assert [(i, r.offsets) for i, r in got] == exp, (m, off)


def test_multi_singleton_equals_sequential(gpu):
    rng = np.random.default_rng(5)
    for _ in range(40):
        text = rng.choice(list(b"ACGT"), int(rng.integers(1, 3000))).astype(np.uint8).tobytes()
        m = int(rng.integers(1, 40))
        pat = rng.choice(list(b"ACGT"), m).astype(np.uint8).tobytes()
        [(idx, res)] = rk.search_multi(text, rk.PatternSet([pat]))
        assert idx == 0 and res == rk.search_sequential(text, pat)


def test_multi_many_lengths_against_oracle(gpu):
    rng = np.random.default_rng(9)
    text = rng.integers(0, 4, 300000, dtype=np.uint8)
    pats = []
    for m in (1, 3, 7, 16, 24, 25, 31, 32, 33, 64, 65, 90):
        for _ in range(20):
            x = int(rng.integers(0, text.size - m))
            pats.append(text[x : x + m].tobytes())
        pats.append(rng.integers(0, 4, m, dtype=np.uint8).tobytes())
    out = rk.search_multi(text.tobytes(), pats)
    ps, by_len, _ = oracle.pattern_set(pats)
    expect = {}
    for m, idxs in by_len.items():
        for j, offs in oracle.c_search_multi_group(text, [ps[i] for i in idxs]):
            expect[idxs[j]] = offs.tolist()
    for i, r in out:
        assert r.offsets == expect[i], (i, len(ps[i]))


def test_dense_all_a(gpu):
    """Adversarial density (C5 shape): every window matches."""
    torch = _torch()
    for n, m in [(4097, 1), (100000, 4), (65536 + 17, 31), (50000, 32), (70000, 100)]:
        t = torch.full((n,), 97, dtype=torch.uint8, device="cuda")
        st = rk.ScanStats()
        offs, k, coll, hits = _scan.scan_counts(t, b"a" * m, rk.hash_full(b"a" * m), 0, n - m + 1)
        assert k == n - m + 1 and coll == 0 and hits == k
        assert torch.equal(offs, torch.arange(n - m + 1, device="cuda")), (n, m)
        r = rk.search_sequential(b"a" * n, b"a" * m, stats=st)
        assert r.offsets == list(range(n - m + 1))
        assert st.collisions == 0


def test_host_overflow_fetch_path(gpu):
    # more matches than the initial capacity of the host path: fetched, never rescanned
    n = (1 << 16) * 3 + 11
    r = rk.search_sequential(b"ab" * (n // 2), b"ab")
    assert r.offsets == list(range(0, 2 * (n // 2) - 1, 2))


def test_search_parallel_devices_kw(gpu):
    rng = np.random.default_rng(1)
    text = rng.integers(0, 4, 100000, dtype=np.uint8).tobytes()
    pat = text[5000:5012]
    cfg = rk.plan_launch(len(text), len(pat), 256)
    r1 = rk.search_parallel(text, pat, cfg, 4, devices=[0])
    assert r1 == rk.search_naive(text, pat)


def test_pinned_host_tensor_input(gpu):
    torch = _torch()
    rng = np.random.default_rng(2)
    host = torch.from_numpy(rng.integers(0, 4, 1 << 20, dtype=np.uint8)).pin_memory()
    pat = host[4321 : 4321 + 20].numpy().tobytes()
    r = rk.search_sequential(host, pat)
    eo, _ = oracle.c_scan(host.numpy(), np.frombuffer(pat, dtype=np.uint8), workers=4)
    assert r.offsets == eo.tolist()


def test_multi_qgram_modes_edges(gpu):
    """q-gram sampled filter (m >= 7): occurrences at both text ends, at every alignment,
    device views at odd offsets, many patterns sharing q-grams."""
    torch = _torch()
    rng = np.random.default_rng(77)
    cases = [(m, 4) for m in (7, 8, 10, 11, 14, 15, 16, 17, 22, 23, 24, 33, 64, 100)]
    cases += [(m, 256) for m in (7, 10, 11, 14, 15, 16, 23, 40)]
    for m, alpha in cases:
        n = 50000
        base = rng.integers(0, alpha, n + 40, dtype=np.uint8)
        for shift in (0, 1, 5, 13):
            host = base[shift : shift + n].copy()
            pats = []
            for x in (0, 1, 2, 3, 7, 8, 9, 4095, 4096, 8191, 8192, n // 2 + 3, n - m - 1, n - m):
                pats.append(host[x : x + m].tobytes())
            for _ in range(40):
                pats.append(rng.integers(0, alpha, m, dtype=np.uint8).tobytes())
            dev = torch.from_numpy(base).cuda()[shift : shift + n]
            out = rk.search_multi(dev, pats)
            ps, by_len, _ = oracle.pattern_set(pats)
            expect = {j: offs.tolist() for j, offs in oracle.c_search_multi_group(host, ps)}
            for i, r in out:
                assert r.offsets == expect[i], (m, shift, i)


def test_multi_mixed_lengths_one_sweep(gpu):
    """Every length >= 7 of a set shares a sweep (64 lengths per launch); lengths < 7 get
    their own; results equal the per-length oracle, at both text ends and any alignment."""
    torch = _torch()
    from paper_1810_01051_b200 import _lib

    rng = np.random.default_rng(81)
    for alpha in (4, 95):
        n = 150000
        base = (rng.integers(0, alpha, n + 16, dtype=np.uint8) + (0 if alpha == 4 else 32)).astype(np.uint8)
        for shift in (0, 3):
            host = base[shift : shift + n].copy()
            lengths = list(range(7, 27)) + [3, 5, 40, 64, 100]
            pats = []
            for m in lengths:
                for x in (0, 1, 4095, 4096, n // 3, n - m):
                    pats.append(host[x : x + m].tobytes())
                pats.append((rng.integers(0, alpha, m) + (0 if alpha == 4 else 32)).astype(np.uint8).tobytes())
            dev = torch.from_numpy(base).cuda()[shift : shift + n]
            ctx = _lib.context()
            before = ctx.launches
            out = rk.search_multi(dev, pats)
            sweeps = ctx.launches - before
            assert sweeps == 2 + 1, sweeps  # m = 3 and 5 alone, the 23 lengths >= 7 in one sweep
            ps, by_len, _ = oracle.pattern_set(pats)
            expect = {}
            for m, idxs in by_len.items():
                for j, offs in oracle.c_search_multi_group(host, [ps[i] for i in idxs]):
                    expect[idxs[j]] = offs.tolist()
            for i, r in out:
                assert r.offsets == expect[i], (alpha, shift, i, len(ps[i]))


def test_multi_mixed_lengths_longer_than_text(gpu):
    """Lengths longer than the text share the sweep with an empty window range."""
    rng = np.random.default_rng(82)
    for n in (7, 40, 100, 5000):
        text = rng.integers(0, 3, n, dtype=np.uint8).tobytes()
        pats = [text[: min(n, m)] if m <= n else bytes(m) for m in range(7, 130, 3)]
        pats += [text[n // 2 : n // 2 + 9], text[-8:]]
        out = rk.search_multi(text, pats)
        ps, _, _ = oracle.pattern_set(pats)
        for i, r in out:
            assert r == rk.search_naive(text, ps[i]), (n, i, len(ps[i]))


def test_multi_pair_counts_at_the_small_sort_limit(gpu):
    """Pair counts around the one-block sort's limit (4096 pairs: kSmallSort) and the
    radix sort above it: planted copies of two patterns in random order, every list exact
    and ascending, for 2, 4095, 4096, 4097 and 9000 pairs."""
    rng = np.random.default_rng(84)
    n = 1 << 20
    for total in (2, 4095, 4096, 4097, 9000):
        text = rng.integers(ord("a"), ord("z") + 1, n, dtype=np.uint8)
        starts = np.sort(rng.choice(n // 16 - 1, total, replace=False)) * 16
        for j, x in enumerate(starts):
            text[x:x + 8] = np.frombuffer(b"QRSTUVWX" if j % 3 else b"QRSTUVWY", np.uint8)
        pats = [b"QRSTUVWX", b"QRSTUVWY", b"ZZZZZZZZZ"]
        out = rk.search_multi(text.tobytes(), pats)
        ps, _, _ = oracle.pattern_set(pats)
        got = 0
        for i, r in out:
            exp = rk.search_naive(text.tobytes(), ps[i])
            assert r == exp, (total, i)
            got += len(r.offsets)
        assert got == total


def test_multi_many_pairs_device_sorted(gpu):
    """More pairs than one block sorts (4096): ordered by the device radix sort."""
    rng = np.random.default_rng(83)
    text = rng.integers(0, 2, 300000, dtype=np.uint8).tobytes()
    pats = [bytes(rng.integers(0, 2, m, dtype=np.uint8)) for m in (3, 5, 8, 8, 9, 12, 20)]
    out = rk.search_multi(text, pats)
    ps, _, _ = oracle.pattern_set(pats)
    total = 0
    for i, r in out:
        exp = rk.search_naive(text, ps[i])
        assert r == exp, i
        total += len(exp.offsets)
    assert total > 20000


def test_multi_plan_cache_keys_on_bytes(gpu):
    """The per-context plan cache must not confuse sets that differ only in pattern bytes
    (equal lengths and hashes: "ac" / "ba", tests/test_matcher.py:139-146 of the reference)."""
    text = b"xacbaacxbaba" * 50
    for pats in (["ac"], ["ba"], ["ac"], ["acbaacxb", "baacxbab"], ["baacxbab", "acbaacxb"]):
        out = rk.search_multi(text, [p.encode() if isinstance(p, str) else p for p in pats])
        for i, r in out:
            assert r == rk.search_naive(text, pats[i].encode()), (pats, i)


def test_multi_4096_patterns(gpu):
    rng = np.random.default_rng(78)
    text = rng.integers(0, 256, 1 << 20, dtype=np.uint8)
    pats = [text[x : x + 16].tobytes() for x in rng.integers(0, (1 << 20) - 16, 3000)]
    pats += [rng.integers(0, 256, 16, dtype=np.uint8).tobytes() for _ in range(1096)]
    out = rk.search_multi(text.tobytes(), pats)
    ps, _, _ = oracle.pattern_set(pats)
    expect = {j: offs.tolist() for j, offs in oracle.c_search_multi_group(text, ps)}
    assert len(out) == len(ps)
    for i, r in out:
        assert r.offsets == expect[i]


def test_bitmap_output(gpu):
    """rk_scan_bitmap == MatchResult.to_bitmap of the oracle offsets (ranges, alignments,
    dense text)."""
    torch = _torch()
    rng = np.random.default_rng(91)
    base = rng.integers(0, 3, 100000, dtype=np.uint8)
    dev_base = torch.from_numpy(base).cuda()
    for shift in (0, 3, 17):
        host = base[shift:]
        dev = dev_base[shift:]
        for m in (1, 4, 9, 31, 32, 40, 70):
            pat = host[5000 : 5000 + m]
            hx = oracle.hash_full(pat.tobytes())
            nw = host.size - m + 1
            for start, stop in [(0, nw), (7, 70000), (33, 34), (nw - 5, nw)]:
                eo, ec = oracle.c_scan(host, pat, start, stop)
                expect = np.zeros(stop - start, dtype=bool)
                expect[eo - start] = True
                bits, k, coll, hits = _scan.scan_bitmap(dev, pat.tobytes(), hx, start, stop)
                assert torch.equal(bits.cpu(), torch.from_numpy(expect)), (shift, m, start, stop)
                assert k == len(eo) and coll == ec and hits == k + coll
                hbits, k2, _, _ = _scan.scan_bitmap(host, pat.tobytes(), hx, start, stop)
                assert (hbits == expect).all() and k2 == k
    # dense: every window
    n = 1 << 20
    t = torch.full((n,), 97, dtype=torch.uint8, device="cuda")
    bits, k, coll, _ = _scan.scan_bitmap(t, b"aaaa", rk.hash_full(b"aaaa"), 0, n - 3)
    assert k == n - 3 and bool(bits.all()) and bits.numel() == n - 3
    st = rk.ScanStats()
    bm = rk.search_bitmap(b"abab", b"ab", stats=st)
    assert bm.tolist() == rk.MatchResult(4, 2, [0, 2]).to_bitmap().tolist()
    assert st == rk.ScanStats(3, 2, 0)


def test_search_each_host_batch(gpu):
    """search_each (rk_scan_host_batch: the host text crosses PCIe once) equals
    search_sequential per pattern, with duplicates, lengths > n, a pattern whose hash no
    window can reach, dense patterns overflowing their first slot, and stats."""
    rng = np.random.default_rng(17)
    n = (130 << 20) + 12345  # 3 staging chunks, ragged
    text = rng.integers(0, 4, n, dtype=np.uint8)
    text[5 << 20: (5 << 20) + 300000] = 0  # a dense run: 'AAAA'-style overflow
    pats = [text[x:x + m].tobytes() for x, m in ((1000, 4), (77777, 8), (3 << 20, 16),
                                                  (100 << 20, 32), (129 << 20, 1024))]
    pats += [bytes(4), pats[1], b"\xff" * 20, bytes(range(200, 230)), b"x" * (n + 1)]
    st = rk.ScanStats()
    got = rk.search_each(text, pats, stats=st)
    st2 = rk.ScanStats()
    for p, r in zip(pats, got):
        e = rk.search_sequential(text, p, stats=st2)
        assert r == e, len(p)
    assert (st.windows, st.hash_hits, st.collisions) == (st2.windows, st2.hash_hits, st2.collisions)
    assert len(got[5].offsets) > (1 << 16)  # the overflowing pattern
    # pageable bytes and a pinned tensor view take the same path
    import torch

    pinned = torch.from_numpy(text).pin_memory()
    assert rk.search_each(pinned.numpy(), pats[:3]) == got[:3]
    assert rk.search_each(text.tobytes()[: 1 << 20], [pats[0]]) == \
        [rk.search_sequential(text.tobytes()[: 1 << 20], pats[0])]


def test_multi_short_lengths_folded(gpu):
    """Every length < 7 of a set in at most two sweeps (1..3 per-window keys, 4..6 anchored
    q-grams, one cuckoo table keyed by (bytes, length) each) next to the >= 7 sweep;
    results equal the per-length oracle at both text ends and at odd device offsets."""
    torch = _torch()
    from paper_1810_01051_b200 import _lib

    rng = np.random.default_rng(91)
    for alpha, lo in ((4, 65), (95, 32), (256, 0)):
        n = 200000
        base = (rng.integers(0, alpha, n + 8, dtype=np.uint8) + lo).astype(np.uint8)
        for shift in (0, 5):
            host = base[shift: shift + n].copy()
            pats = []
            for m in (1, 2, 3, 4, 5, 6, 9, 20):
                for x in (0, 1, 1023, 1024, 4095, n // 2, n - m):
                    pats.append(host[x: x + m].tobytes())
                for _ in range(30):
                    pats.append((rng.integers(0, alpha, m) + lo).astype(np.uint8).tobytes())
            dev = torch.from_numpy(base).cuda()[shift: shift + n]
            ctx = _lib.context()
            before = ctx.launches
            out = rk.search_multi(dev, pats)
            total = sum(len(r.offsets) for _, r in out)
            # 1..3, 4..6, >= 7 (twice when the pairs overflow search_multi's first buffer)
            assert ctx.launches - before == 3 * (2 if total > max(1 << 16, n) else 1)
            ps, by_len, _ = oracle.pattern_set(pats)
            expect = {}
            for m, idxs in by_len.items():
                for j, offs in oracle.c_search_multi_group(host, [ps[i] for i in idxs]):
                    expect[idxs[j]] = offs.tolist()
            for i, r in out:
                assert r.offsets == expect[i], (alpha, shift, i, len(ps[i]))


def test_multi_dense_short_lengths(gpu):
    """Dense output through the short sweeps: all 'a' against a, aa, ..., a^8 -- every
    window of every length matches (appended one atomic per warp per round)."""
    torch = _torch()
    for n in (200003, 4096 + 7):
        t = torch.full((n,), 97, dtype=torch.uint8, device="cuda")
        pats = [b"a" * m for m in range(1, 9)] + [b"ab", b"aab", b"aaaab"]
        out = rk.search_multi(t, pats)
        for i, r in out:
            m = len(pats[i])
            exp = list(range(n - m + 1)) if b"b" not in pats[i] else []
            assert r.offsets == exp, (n, pats[i])


def test_search_parallel_device_shards_host_text(gpu):
    """search_parallel(devices=[...]) with a host text: each shard goes through its device's
    own staging pipeline (here two shards on cuda:0, scanned concurrently on two contexts)
    and the rank-order concatenation equals the reference's result; pageable and pinned."""
    torch = _torch()
    rng = np.random.default_rng(12)
    text = rng.integers(0, 4, (3 << 20) + 11, dtype=np.uint8)
    for pat in (text[1000:1008].tobytes(), text[(3 << 20) // 2 - 4:(3 << 20) // 2 + 28].tobytes()):
        cfg = rk.plan_launch(text.size, len(pat), 256)
        st = rk.ScanStats()
        r = rk.search_parallel(text.tobytes(), pat, cfg, 4, stats=st, devices=[0, 0])
        st2 = rk.ScanStats()
        assert r == rk.search_sequential(text.tobytes(), pat, stats=st2)
        assert (st.hash_hits, st.collisions) == (st2.hash_hits, st2.collisions)
        pinned = torch.from_numpy(text).pin_memory()
        assert rk.search_parallel(pinned.numpy(), pat, cfg, 2, devices=[0, 0]) == r


def test_search_each_many_patterns(gpu):
    """More patterns than one rk_scan_host_batch call takes (64): split into batches, each
    staging the text once; results and stats equal search_sequential's; no patterns: []."""
    rng = np.random.default_rng(18)
    text = rng.integers(0, 4, (5 << 20) + 3, dtype=np.uint8)
    pats = [text[x:x + m].tobytes() for x, m in zip(rng.integers(0, text.size - 64, 70),
                                                     rng.integers(1, 64, 70))]
    st = rk.ScanStats()
    got = rk.search_each(text.tobytes(), pats, stats=st)
    st2 = rk.ScanStats()
    assert got == [rk.search_sequential(text.tobytes(), p, stats=st2) for p in pats]
    assert (st.windows, st.hash_hits, st.collisions) == (st2.windows, st2.hash_hits, st2.collisions)
    assert rk.search_each(text.tobytes(), []) == []
    with pytest.raises(ValueError):
        rk.search_each(text.tobytes(), [b"ab", b""])
