"""Host-side logic of the drop-in API (no GPU): hashing, PatternSet, launch algebra,
validation order and exception types -- mirrored from the reference's own tests
(/root/reference/pkg/tests/test_rkhash.py, test_matcher.py, test_parallel.py) and
checked against the golden vectors."""

import itertools
import random

import numpy as np
import pytest

import paper_1810_01051_b200 as rk
from paper_1810_01051_b200 import _scan
from tests import _golden as G


def test_hash_full_golden():
    for e in G.hash_kat()["hash_full"]:
        assert rk.hash_full(G.dec(e["data"])) == int(e["h"])


def test_hash_examples():
    assert rk.hash_full(b"") == 0
    assert rk.hash_full(b"a") == 97
    assert rk.hash_full(b"ab") == 292
    assert rk.hash_full(b"ac") == rk.hash_full(b"ba") == 293
    assert rk.hash_full(bytearray(b"acgt")) == rk.hash_full(memoryview(b"acgt"))
    assert rk.hash_full(b"\xff" + b"q" * 64) == rk.hash_full(b"\x00" + b"q" * 64)
    assert rk.hash_full(b"q\xff" + b"q" * 63) != rk.hash_full(b"q\x00" + b"q" * 63)
    assert 0 <= rk.hash_full(b"\xff" * 4096) <= rk.MASK64


def test_hash_window_and_roll():
    for e in G.hash_kat()["hash_window"]:
        assert rk.hash_window(G.dec(e["text"]), e["off"], e["m"]) == int(e["h"])
    for e in G.hash_kat()["roll"]:
        assert rk.roll(int(e["prev"]), e["out"], e["in"], e["m"]) == int(e["h"])
    with pytest.raises(ValueError):
        rk.hash_window(b"abc", 2, 2)
    with pytest.raises(ValueError):
        rk.hash_window(b"abc", -1, 2)
    with pytest.raises(ValueError):
        rk.hash_window(b"abc", 0, 0)
    with pytest.raises(ValueError):
        rk.roll(0, 0, 0, 0)


def test_hash_window_exhaustive_small_alphabet():
    for n in range(1, 6):
        for text in itertools.product(b"ab", repeat=n):
            text = bytes(text)
            for m in range(1, n + 1):
                for x in range(n - m + 1):
                    assert rk.hash_window(text, x, m) == rk.hash_full(text[x : x + m])


def test_as_u8():
    with pytest.raises(TypeError):
        _scan.as_u8("text")
    with pytest.raises(TypeError):
        _scan.as_u8(np.zeros(4, dtype=np.int32))
    assert _scan.as_u8(b"ab").dtype == np.uint8
    import torch

    with pytest.raises(TypeError):
        _scan.as_u8(torch.zeros(4, dtype=torch.int32))
    assert _scan.as_u8(torch.zeros(4, dtype=torch.uint8)).dtype == torch.uint8


def test_pattern_set():
    ps = rk.PatternSet([b"ab", b"ba", b"a", b"ab"])
    assert ps.patterns == [b"ab", b"ba", b"a"]
    assert ps.by_length == {2: [0, 1], 1: [2]}
    assert ps.hash_index[2] == {292: [0], 293: [1]}
    assert len(ps) == 3
    with pytest.raises(ValueError):
        rk.PatternSet([])
    with pytest.raises(ValueError):
        rk.PatternSet([b"ok", b""])
    for c in G.multi_cases():
        assert rk.PatternSet(c["patterns"]).patterns == c["deduped"]


def test_match_result_bitmap():
    r = rk.MatchResult(4, 2, [0, 2])
    assert r.to_bitmap().tolist() == [True, False, True]
    assert rk.MatchResult(2, 3, []).to_bitmap().size == 0


def test_search_naive_examples():
    assert rk.search_naive(b"abab", b"ab").offsets == [0, 2]
    assert rk.search_naive(b"aaaa", b"aa").offsets == [0, 1, 2]
    assert rk.search_naive(b"ab", b"abc").offsets == []
    with pytest.raises(ValueError):
        rk.search_naive(b"abc", b"")


def test_launch_algebra_golden():
    L = G.launch()
    for e in L["plan"]:
        cfg = rk.plan_launch(e["n"], e["m"], e["block"], e["cap"])
        assert list(cfg.grid_dims) == e["grid"] and cfg.total_threads == e["total"]
    for e in L["offset_of"]:
        cfg = rk.LaunchConfig(tuple(e["grid"]), e["block"])
        assert rk.offset_of(rk.ThreadCoord(tuple(e["block_idx"]), e["thread"]), cfg) == e["offset"]


def test_offset_of_bijective():
    for dims in itertools.product((1, 2, 3), repeat=3):
        for block_dim in (1, 7, 32):
            cfg = rk.LaunchConfig(dims, block_dim)
            seen = set()
            gx, gy, gz = dims
            for bz, by, bx in itertools.product(range(gz), range(gy), range(gx)):
                for t in range(block_dim):
                    seen.add(rk.offset_of(rk.ThreadCoord((bx, by, bz), t), cfg))
            assert seen == set(range(cfg.total_threads))


def test_launch_validation():
    with pytest.raises(ValueError):
        rk.LaunchConfig((0, 1, 1), 32)
    with pytest.raises(ValueError):
        rk.LaunchConfig((1, 1, 1), 0)
    with pytest.raises(ValueError):
        rk.LaunchConfig((1, 1, 1), 1025)
    assert rk.LaunchConfig((2, 3, 4), 5).total_threads == 120
    for args in [(10, 11, 32), (10, 2, 0), (10, 2, 1025), (10, 0, 32)]:
        with pytest.raises(ValueError):
            rk.plan_launch(*args)
    cfg = rk.LaunchConfig((2, 2, 2), 8)
    for coord in [((2, 0, 0), 0), ((0, -1, 0), 0), ((0, 0, 0), 8)]:
        with pytest.raises(ValueError):
            rk.offset_of(rk.ThreadCoord(*coord), cfg)


def test_plan_launch_covers_all_windows():
    rng = random.Random(17)
    for _ in range(200):
        n = rng.randrange(1, 100_000)
        m = rng.randrange(1, n + 1)
        b = rng.choice((1, 32, 256, 1024))
        cfg = rk.plan_launch(n, m, b)
        assert cfg.total_threads >= n - m + 1


def test_hash_pattern_host():
    assert rk.hash_pattern_host(b"ab") == 292
    assert rk.hash_pattern_host(b"ba") == 293
    with pytest.raises(ValueError):
        rk.hash_pattern_host(b"")


def test_search_validation_before_device():
    """Errors the reference raises before scanning are raised before touching the GPU
    (parallel.py:140-153, matcher.py:108-115): they hold on a machine with no device."""
    with pytest.raises(ValueError):
        rk.search_parallel(b"abcdef", b"ab", rk.LaunchConfig((1, 1, 1), 2), workers=1)
    with pytest.raises(ValueError):
        rk.search_parallel(b"abab", b"", rk.plan_launch(4, 1, 32), workers=1)
    with pytest.raises(ValueError):
        rk.search_parallel(b"abab", b"ab", rk.plan_launch(4, 2, 32), workers=0)
    with pytest.raises(TypeError):
        rk.search_parallel("abab", b"ab", rk.plan_launch(4, 2, 32))
    with pytest.raises(ValueError):
        rk.search_sequential(b"abc", b"")
    with pytest.raises(TypeError):
        rk.search_sequential("abc", b"a")
    # no windows: empty result, stats untouched, no device needed
    st = rk.ScanStats()
    r = rk.search_sequential(b"ab", b"abc", stats=st)
    assert r == rk.MatchResult(2, 3, []) and st == rk.ScanStats()
    r = rk.search_parallel(b"ab", b"abc", rk.LaunchConfig((1, 1, 1), 1), workers=3)
    assert r.offsets == []
    out = rk.search_multi(b"ab", rk.PatternSet([b"abcd"]))
    assert [(i, x.offsets) for i, x in out] == [(0, [])]


def test_splitmix_golden():
    co = G.corpus()
    state = 0
    for v in co["splitmix64_seed0_chain"]:
        out, state = rk.splitmix64(state)
        assert out == int(v)
    assert rk.splitmix64_stream(42, 16, 1000).tolist() == [
        int(v) for v in co["stream_seed42_skip1000"]
    ]


def test_plant():
    assert rk.plant(b"xxxxxx", b"ab", [0, 3]) == b"abxabx"
    with pytest.raises(ValueError):
        rk.plant(b"xxxx", b"ab", [0, 1])
    with pytest.raises(ValueError):
        rk.plant(b"xxxx", b"ab", [3])
    with pytest.raises(ValueError):
        rk.plant(b"xxxx", b"", [0])


def test_shard_ranges_cover_exactly_once():
    from paper_1810_01051_b200.parallel import shard_ranges

    for W in (1, 2, 7, 100, 4097):
        for G_ in (1, 2, 3, 4, 8):
            r = shard_ranges(W, G_)
            covered = [x for a, b in r for x in range(a, b)]
            assert covered == list(range(W))


def test_acceptance_criterion5_host_roll(golden):
    """The reference's criterion 5 (test_acceptance.py:156-182) on the host hash
    functions: rolling every window of the 1,000 texts with rk.roll tracks
    rk.hash_window, and the chain's digest is the reference's."""
    import numpy as np

    for j, (text, m, dig) in enumerate(golden.criterion5_texts()):
        h = rk.hash_window(text, 0, m)
        chain = [h]
        for x in range(len(text) - m):
            h = rk.roll(h, text[x], text[x + m], m)
            chain.append(h)
        if j % 25 == 0:
            assert chain[-1] == rk.hash_window(text, len(text) - m, m)
        assert golden.digest(chain, np.uint64) == dig
    c = golden.acceptance()["criterion5_m65"]
    base = golden.dec(c["base"])
    variant = bytes([base[0] ^ 0xFF]) + base[1:]
    assert rk.hash_window(base, 0, 65) == rk.hash_window(variant, 0, 65) == int(c["h"])
    h = rk.hash_window(base, 0, 65)
    for x in range(len(base) - 65):
        h = rk.roll(h, base[x], base[x + 65], 65)
        assert h == rk.hash_window(base, x + 1, 65)
