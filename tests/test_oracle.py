"""Pin the CPU oracle (oracle/) to the golden vectors the reference produced.

The oracle is the checker for every GPU parity test, so it must itself agree with the
reference on every fixture: hash known answers, window hashes, single-pattern cases
(offsets + windows + hash_hits + collisions), corpus checksums, the C1 / 1 MiB length
sweep, DNA with planted copies, and search_multi cases.
"""

import hashlib

import numpy as np
import pytest

import oracle
from tests import _golden as G


def test_hash_known_answers():
    kat = G.hash_kat()
    for e in kat["hash_full"]:
        data = G.dec(e["data"])
        assert oracle.hash_full(data) == int(e["h"])
        lib = oracle.load()
        buf = np.frombuffer(data, dtype=np.uint8)
        assert lib.ro_hash_full(buf.ctypes.data if data else 0, len(data)) == int(e["h"])
    for e in kat["hash_window"]:
        assert oracle.hash_window(G.dec(e["text"]), e["off"], e["m"]) == int(e["h"])
    for e in kat["roll"]:
        assert oracle.roll(int(e["prev"]), e["out"], e["in"], e["m"]) == int(e["h"])


def test_window_hashes_numpy_and_c():
    for e in G.hash_kat()["window_hashes"]:
        text = np.frombuffer(G.dec(e["text"]), dtype=np.uint8)
        m = e["m"]
        expect = [int(v) for v in e["h"]]
        stop = text.size - m + 1
        assert oracle.window_hashes(text, m, 0, stop).tolist() == expect
        assert oracle.c_window_hashes(text, m, 0, stop).tolist() == expect


def test_scan_cases_c_oracle():
    cases = G.scan_cases()
    assert len(cases) > 400
    for c in cases:
        t = np.frombuffer(c["text"], dtype=np.uint8)
        p = np.frombuffer(c["pattern"], dtype=np.uint8)
        offs, coll = oracle.c_scan(t, p)
        assert offs.tolist() == c["offsets"], c["tag"]
        assert coll == c["collisions"], c["tag"]
        assert len(offs) + coll == c["hash_hits"], c["tag"]


def test_scan_cases_numpy_oracle_and_parallel_c():
    for i, c in enumerate(G.scan_cases()):
        if i % 3:
            continue
        n, m, offs, stats = oracle.search_sequential(c["text"], c["pattern"])
        assert offs == c["offsets"], c["tag"]
        assert stats["collisions"] == c["collisions"]
        assert stats["hash_hits"] == c["hash_hits"]
        assert stats["windows"] == c["windows"]
        if c["m"] <= c["n"]:
            t = np.frombuffer(c["text"], dtype=np.uint8)
            p = np.frombuffer(c["pattern"], dtype=np.uint8)
            po, pc = oracle.c_scan(t, p, workers=4)
            assert po.tolist() == c["offsets"] and pc == c["collisions"], c["tag"]


def test_naive_agrees_on_small_cases():
    for c in G.scan_cases()[:60]:
        if c["m"] <= c["n"] or c["n"] == 0:
            assert oracle.search_naive(c["text"], c["pattern"]) == c["offsets"], c["tag"]


def test_corpus_checksums_and_streams():
    co = G.corpus()
    state = 0
    for v in co["splitmix64_seed0_chain"]:
        out, state = oracle.splitmix64(state)
        assert out == int(v)
    assert oracle.splitmix64_stream(42, 16, 1000).tolist() == [
        int(v) for v in co["stream_seed42_skip1000"]
    ]
    dna = oracle.generate(42, 2 * 2**20)
    assert hashlib.sha256(dna).hexdigest() == co["dna_seed42_2MiB_sha256"]
    a1 = oracle.generate(42, 2**20, G.ASCII)
    assert hashlib.sha256(a1).hexdigest() == co["ascii_seed42_1MiB_sha256"]
    a3 = oracle.generate(43, 2**20, G.ASCII)
    assert hashlib.sha256(a3).hexdigest() == co["ascii_seed43_1MiB_sha256"]


def test_c1_sweep_1mib():
    co = G.corpus()
    text = oracle.generate(42, 2**20, G.ASCII)
    t = np.frombuffer(text, dtype=np.uint8)
    for e in co["ascii_seed42_1MiB_sweep"]:
        pat = G.dec(e["pattern"])
        assert pat == oracle.make_pattern(text, 42, G.ASCII, e["m"], e["source"])
        offs, coll = oracle.c_scan(t, np.frombuffer(pat, dtype=np.uint8),
                                   workers=oracle.cpu_threads())
        assert offs.tolist() == e["offsets"], (e["m"], e["source"])
        assert coll == e["collisions"], (e["m"], e["source"])
        assert len(offs) + coll == e["hash_hits"]


def test_dna_planted_4mib():
    co = G.corpus()
    dna = oracle.generate(42, 4 * 2**20)
    assert hashlib.sha256(dna).hexdigest() == co["dna_seed42_4MiB_sha256"]
    for e in co["dna_seed42_4MiB"]:
        pat = G.dec(e["pattern"])
        text = oracle.plant(dna, pat, e["plant"])
        offs, coll = oracle.c_scan(np.frombuffer(text, dtype=np.uint8),
                                   np.frombuffer(pat, dtype=np.uint8), workers=4)
        assert offs.tolist() == e["offsets"]
        assert coll == e["collisions"]


def test_multi_cases():
    for c in G.multi_cases():
        got = oracle.search_multi(c["text"], c["patterns"])
        assert [[i, o] for i, o in got] == c["results"], c["tag"]
        pats, _, _ = oracle.pattern_set(c["patterns"])
        assert pats == c["deduped"]
        # the C restatement per equal-length group
        t = np.frombuffer(c["text"], dtype=np.uint8)
        expect = dict((i, o) for i, o in c["results"])
        by_len = {}
        for i, p in enumerate(pats):
            by_len.setdefault(len(p), []).append(i)
        for m, idxs in by_len.items():
            if m > t.size:
                continue
            for (j, offs) in oracle.c_search_multi_group(t, [pats[i] for i in idxs]):
                assert offs.tolist() == expect[idxs[j]], (c["tag"], m)


def test_launch_algebra():
    L = G.launch()
    for e in L["plan"]:
        grid, block = oracle.plan_launch(e["n"], e["m"], e["block"], e["cap"])
        assert list(grid) == e["grid"]


@pytest.mark.parametrize("m", [1, 4, 31, 32, 33, 64, 65, 200])
def test_roll_matches_window_hashes(m):
    rng = np.random.default_rng(m)
    t = rng.integers(0, 256, 700, dtype=np.uint8)
    h = oracle.window_hashes(t, m, 0, t.size - m + 1)
    cur = int(h[0])
    for x in range(t.size - m):
        cur = oracle.roll(cur, int(t[x]), int(t[x + m]), m)
        assert cur == int(h[x + 1])


# --------------------------------------------------------------------------- acceptance
def test_acceptance_criterion1_c_oracle(golden):
    """All 10,008 cases of the reference's criterion 1 (test_acceptance.py:49-85): the C
    oracle (per-window and rolled, parallel partition included) gives the reference's
    recorded offsets and collision counts."""
    import numpy as np

    n_cases = 0
    for case, text, pattern, workers, block, exp in golden.criterion1_cases():
        n, m = len(text), len(pattern)
        t = np.frombuffer(text, dtype=np.uint8)
        p = np.frombuffer(pattern, dtype=np.uint8)
        if m > n:
            assert exp[3] == 0 and exp[4] == 0
            continue
        eo, ec = oracle.c_scan(t, p)
        assert (eo.size, ec, golden.digest(eo, np.int64)) == tuple(exp[3:]), case
        if case % 4 == 0:
            ro, rc = oracle.c_scan_mt(t, pattern, threads=workers)
            assert ro.size == eo.size and (ro == eo).all() and rc == ec, case
        n_cases += 1
    assert n_cases > 9000


def test_acceptance_criterion4_collision_family(golden):
    """Criterion 4 (test_acceptance.py:124-153) with the oracle: byte-true offsets and the
    reference's collision counts; the verify-fail branch is taken."""
    import numpy as np

    filler = oracle.generate(11, 5000)
    texts = [b"ac" + b"Xba" * 300, oracle.plant(filler, b"ba", list(range(0, 4000, 13))),
             b"ba" * 64 + b"ac" + b"ba" * 64]
    total = 0
    for c in golden.acceptance()["criterion4"]:
        text, pat = texts[c["text"]], c["pattern"].encode()
        eo, ec = oracle.c_scan(np.frombuffer(text, np.uint8), np.frombuffer(pat, np.uint8))
        assert eo.tolist() == c["offsets"] == oracle.search_naive(text, pat)
        assert ec == c["collisions"] and c["hash_hits"] == len(c["offsets"]) + ec
        total += ec
    assert total > 0


def test_acceptance_criterion5_rolling(golden):
    """Criterion 5 (test_acceptance.py:156-182): the oracle's batched window hashes give
    the reference's recorded digests for all 1,000 texts, and the m = 65 horizon case."""
    import numpy as np

    for text, m, dig in golden.criterion5_texts():
        t = np.frombuffer(text, dtype=np.uint8)
        assert golden.digest(oracle.c_window_hashes(t, m, 0, t.size - m + 1), np.uint64) == dig
    c = golden.acceptance()["criterion5_m65"]
    base = golden.dec(c["base"])
    variant = bytes([base[0] ^ 0xFF]) + base[1:]
    assert oracle.hash_window(base, 0, 65) == oracle.hash_window(variant, 0, 65) == int(c["h"])
