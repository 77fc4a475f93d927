"""Generate the golden fixtures in tests/golden/ by running the REFERENCE itself.

Run in the build container (the only place /root/reference exists):

    python tests/golden/make_golden.py

The reference package is imported from a scratch copy under /tmp (its numba
``cache=True`` would otherwise write into the read-only tree).  Every expected value in
the fixtures comes from the reference's own public API (``search_sequential``,
``search_parallel``, ``search_multi``, ``ScanStats``, ``window_hashes``, ``generate``,
``_make_pattern``, ``plan_launch``) -- never from this repo's code -- so the fixtures
pin both the oracle (``oracle/``) and the CUDA path.

Output files (JSON; texts are zlib+base64 encoded):
  hash_kat.json    hash_full / hash_window / roll / window_hashes known answers
  scan_cases.json  single-pattern cases: text, pattern, offsets, windows, hash_hits,
                   collisions (seq and par checked equal here before writing)
  corpus.json      splitmix64 chains, corpus sha256s, C1/C2-at-1MiB/DNA goldens
  multi_cases.json search_multi cases
  launch.json      plan_launch / offset_of known answers
  acceptance.json  the reference's acceptance criteria 1, 4, 5 case by case (answers only;
                   inputs are regenerated from the same seeds in tests/_golden.py)
"""

from __future__ import annotations

import base64
import hashlib
import json
import os
import shutil
import sys
import zlib
from pathlib import Path

import numpy as np

OUT = Path(__file__).resolve().parent
REF_SRC = Path("/root/reference/pkg")
SCRATCH = Path("/tmp/rk_golden_ref")


def _import_reference():
    if SCRATCH.exists():
        shutil.rmtree(SCRATCH)
    shutil.copytree(REF_SRC, SCRATCH / "pkg")
    os.environ["NUMBA_CACHE_DIR"] = str(SCRATCH / "numba_cache")
    sys.dont_write_bytecode = True
    sys.path.insert(0, str(SCRATCH / "pkg" / "src"))
    import rkmatch  # noqa: F401

    return rkmatch


def enc(b: bytes) -> str:
    return base64.b64encode(zlib.compress(bytes(b), 9)).decode("ascii")


def main() -> None:
    rk = _import_reference()
    from rkmatch import _scan
    from rkmatch.bench import _make_pattern

    # ------------------------------------------------------------------ hash KATs
    rng = np.random.default_rng(99)
    kat = {"hash_full": [], "hash_window": [], "roll": [], "window_hashes": []}
    for data in [b"", b"a", b"ab", b"ac", b"ba", b"ACGT", bytes(range(256)), b"\xff" * 4096,
                 b"\xff" + b"q" * 64, b"\x00" + b"q" * 64, b"q\xff" + b"q" * 63,
                 b"q\x00" + b"q" * 63, bytes(rng.integers(0, 256, 1000, dtype=np.uint8))]:
        kat["hash_full"].append({"data": enc(data), "h": str(rk.hash_full(data))})
    for text, off, m in [(b"abab", 0, 2), (b"abab", 2, 2), (b"abab", 1, 2)]:
        kat["hash_window"].append({"text": enc(text), "off": off, "m": m,
                                   "h": str(rk.hash_window(text, off, m))})
    for prev, o, i, m in [(292, 97, 97, 2), (rk.hash_full(b"aa"), 97, 97, 2), (293, 98, 98, 2),
                          (12345678901234567890, 255, 1, 64), (2**64 - 1, 255, 255, 65),
                          (2**63, 200, 7, 1), (1, 255, 0, 33)]:
        kat["roll"].append({"prev": str(prev), "out": o, "in": i, "m": m,
                            "h": str(rk.roll(prev, o, i, m))})
    text = bytes(rng.integers(0, 256, 300, dtype=np.uint8))
    arr = _scan.as_u8(text)
    for m in (1, 2, 7, 31, 32, 33, 63, 64, 65, 100, 255):
        h = _scan.window_hashes(arr, m, 0, len(text) - m + 1)
        kat["window_hashes"].append({"text": enc(text), "m": m, "start": 0,
                                     "h": [str(int(v)) for v in h]})
    (OUT / "hash_kat.json").write_text(json.dumps(kat))

    # ------------------------------------------------------------------ scan cases
    cases = []

    def add(tag, text, pattern, check_par=True):
        text = bytes(text)
        pattern = bytes(pattern)
        st = rk.ScanStats()
        res = rk.search_sequential(text, pattern, stats=st)
        if check_par:
            n, m = len(text), len(pattern)
            if m <= n:
                for block in (32, 1024):
                    cfg = rk.plan_launch(n, m, block)
                    st2 = rk.ScanStats()
                    par = rk.search_parallel(text, pattern, cfg, 4, stats=st2)
                    assert par == res and st2.collisions == st.collisions, tag
        naive = rk.search_naive(text, pattern)
        assert naive == res, tag
        cases.append({"tag": tag, "text": enc(text), "pattern": enc(pattern),
                      "n": len(text), "m": len(pattern), "offsets": res.offsets,
                      "windows": st.windows, "hash_hits": st.hash_hits,
                      "collisions": st.collisions})

    # frozen examples (tests/test_matcher.py:29-70, tests/test_parallel.py:113-185)
    add("abab/ab", b"abab", b"ab")
    add("aaaa/aa", b"aaaa", b"aa")
    add("ab/abc", b"ab", b"abc")
    add("acXba/ac", b"acXba", b"ac")
    add("z/z", b"z", b"z")
    add("empty-text", b"", b"a", check_par=False)
    for n, m in [(1, 1), (5, 2), (64, 63), (100, 1), (37, 37), (4097, 1), (1000, 64), (1000, 65),
                 (3000, 1024)]:
        add(f"uniform-a{n}/a{m}", b"a" * n, b"a" * m)
    add("oversized", b"abcabcabcXabcabc" + b"abc" * 3 + b"c", b"abc")

    # collision family (tests/test_acceptance.py:124-153)
    filler = rk.generate(rk.DnaSpec(seed=11, length=5000))
    for ti, text in enumerate([b"ac" + b"Xba" * 300,
                               rk.plant(filler, b"ba", list(range(0, 4000, 13))),
                               b"ba" * 64 + b"ac" + b"ba" * 64]):
        for pat in (b"ac", b"ba"):
            add(f"collision-family-{ti}/{pat.decode()}", text, pat)

    # crafted collisions across the 32-bit and 64-bit hash boundary.  hash is linear:
    # changing byte i by d changes h by d * 2^(m-1-i) mod 2^64.
    crng = np.random.default_rng(777)
    for m in (2, 3, 8, 16, 24, 25, 31, 32, 33, 40, 63, 64, 65, 66, 100, 200, 1024):
        base = bytearray(crng.integers(40, 200, m, dtype=np.uint8).tobytes())
        pat = bytes(base)
        variants = []
        # (a) "ac" -> "ba" at the tail: equal 64-bit hash, bytes differ -> collision
        v = bytearray(base)
        v[m - 2] = base[m - 2] + 1
        v[m - 1] = base[m - 1] - 2
        if m >= 2:
            variants.append(bytes(v))
        # (b) +1 at coefficient 2^k for k in {32, 40, 63} and compensating -2 at 2^(k-1):
        for k in (32, 40, 63):
            i = m - 1 - k
            if i >= 0:
                v = bytearray(base)
                v[i] += 1
                v[i + 1] -= 2
                variants.append(bytes(v))  # equal hash -> collision
                v = bytearray(base)
                v[i] += 1
                variants.append(bytes(v))  # low 32 equal when k >= 32, high differs -> no hit
        # (c) changes at coefficient >= 2^64 (i < m-64) are invisible -> collision
        if m >= 65:
            v = bytearray(base)
            v[0] ^= 0x55
            variants.append(bytes(v))
        # (d) +2 at coefficient 2^63 == 2^64 == 0 -> collision
        if m >= 64:
            v = bytearray(base)
            v[m - 64] = (v[m - 64] + 2) & 0xFF
            variants.append(bytes(v))
        filler = crng.integers(40, 200, 3 * m + 500, dtype=np.uint8).tobytes()
        pieces = [filler[:97], pat]
        for j, var in enumerate(variants):
            pieces += [filler[j * 7: j * 7 + 13 + j], var]
        pieces += [pat, filler[:31 + m % 17], pat]
        add(f"crafted-m{m}", b"".join(pieces), pat)

    # seeded random cases in the shape of tests/test_acceptance.py:49-85 (subset)
    arng = np.random.default_rng(20240810)
    for case in range(420):
        k = (2, 4, 256)[case % 3]
        n = int(arng.integers(1, 4097))
        m = int(arng.integers(1, 65))
        text = arng.integers(0, k, size=n, dtype=np.uint8).tobytes()
        if m <= n and arng.random() < 0.5:
            x = int(arng.integers(0, n - m + 1))
            pattern = text[x: x + m]
        else:
            pattern = arng.integers(0, k, size=m, dtype=np.uint8).tobytes()
        add(f"accept-{case}", text, pattern, check_par=(case % 7 == 0))

    # large-m, high-byte and mid-size cases
    lrng = np.random.default_rng(4242)
    for m in (65, 100, 127, 128, 129, 255, 256, 511, 513, 800, 1024, 1500):
        n = 6000 + m
        text = bytearray(lrng.integers(0, 256, n, dtype=np.uint8).tobytes())
        pat = bytes(text[1000:1000 + m])
        for x in (0, 2500, n - m):
            text[x:x + m] = pat
        # a collision: differ only before the 64-byte horizon
        y = 4000
        if y + m <= n - m:
            text[y:y + m] = pat
            text[y] ^= 0xA5
        add(f"large-m{m}", bytes(text), pat)
    (OUT / "scan_cases.json").write_text(json.dumps(cases))

    # ------------------------------------------------------------------ corpus + configs
    corpus = {}
    state = 0
    chain = []
    for _ in range(8):
        v, state = rk.splitmix64(state)
        chain.append(str(v))
    corpus["splitmix64_seed0_chain"] = chain
    corpus["stream_seed42_skip1000"] = [str(int(v)) for v in rk.splitmix64_stream(42, 16, 1000)]
    dna2 = rk.generate(rk.DnaSpec(seed=42, length=2 * 2**20))
    corpus["dna_seed42_2MiB_sha256"] = hashlib.sha256(dna2).hexdigest()
    ascii_alpha = bytes(range(32, 127))
    c1spec = rk.DnaSpec(seed=42, length=2**20, alphabet=ascii_alpha)
    c1 = rk.generate(c1spec)
    corpus["ascii_seed42_1MiB_sha256"] = hashlib.sha256(c1).hexdigest()
    corpus["ascii_seed43_1MiB_sha256"] = hashlib.sha256(
        rk.generate(rk.DnaSpec(seed=43, length=2**20, alphabet=ascii_alpha))).hexdigest()
    # C1 and the C2 length sweep at 1 MiB (reference CPU scale)
    sweep = []
    for m in (4, 7, 8, 16, 25, 32, 64, 65, 100, 128, 256, 512, 800, 1024):
        for source in ("sampled", "generated"):
            pat = _make_pattern(c1, c1spec, m, source)
            st = rk.ScanStats()
            res = rk.search_sequential(c1, pat, stats=st)
            sweep.append({"m": m, "source": source, "pattern": enc(pat), "offsets": res.offsets,
                          "hash_hits": st.hash_hits, "collisions": st.collisions,
                          "windows": st.windows})
    corpus["ascii_seed42_1MiB_sweep"] = sweep
    # DNA: m=8 (collision-rich) and m=32 with planted copies, 4 MiB
    dspec = rk.DnaSpec(seed=42, length=4 * 2**20)
    dna = rk.generate(dspec)
    dna_cases = []
    for m in (8, 32):
        pat = _make_pattern(dna, dspec, m, "sampled")
        planted = rk.plant(dna, pat, [2**20 - 16, 2**21 - 16, 3 * 2**20 - 16])
        st = rk.ScanStats()
        res = rk.search_sequential(planted, pat, stats=st)
        dna_cases.append({"m": m, "pattern": enc(pat), "plant": [2**20 - 16, 2**21 - 16,
                                                                   3 * 2**20 - 16],
                          "offsets": res.offsets, "hash_hits": st.hash_hits,
                          "collisions": st.collisions, "windows": st.windows})
    corpus["dna_seed42_4MiB"] = dna_cases
    corpus["dna_seed42_4MiB_sha256"] = hashlib.sha256(dna).hexdigest()
    (OUT / "corpus.json").write_text(json.dumps(corpus))

    # ------------------------------------------------------------------ multi cases
    multi = []

    def addm(tag, text, patterns):
        ps = rk.PatternSet(patterns)
        out = rk.search_multi(text, ps)
        for i, r in out:
            assert r == rk.search_naive(text, ps.patterns[i]), tag
        multi.append({"tag": tag, "text": enc(text), "patterns": [enc(p) for p in patterns],
                      "deduped": [enc(p) for p in ps.patterns],
                      "results": [[i, r.offsets] for i, r in out]})

    addm("abab/ab,ba", b"abab", [b"ab", b"ba"])
    addm("abab/ac", b"abab", [b"ac"])
    addm("aaa/a,aa", b"aaa", [b"a", b"aa"])
    addm("acbaac/ac,ba", b"acbaac", [b"ac", b"ba"])
    addm("ab/abcd,b", b"ab", [b"abcd", b"b"])
    addm("dup", b"abababab", [b"ab", b"ba", b"a", b"ab"])
    addm("blocks", (b"A" * 250 + b"CG") * 40, [b"CG"])
    mrng = np.random.default_rng(6)
    for t in range(40):
        alpha = (b"ab", b"ACGT", bytes(range(256)))[t % 3]
        n = int(mrng.integers(1, 600))
        text = bytes(mrng.choice(list(alpha), n).astype(np.uint8))
        pats = []
        for _ in range(int(mrng.integers(1, 12))):
            m = int(mrng.integers(1, 9))
            if n >= m and mrng.random() < 0.5:
                x = int(mrng.integers(0, n - m + 1))
                pats.append(text[x:x + m])
            else:
                pats.append(bytes(mrng.choice(list(alpha), m).astype(np.uint8)))
        addm(f"rand-{t}", text, pats)
    # C3 shape at reduced scale: 1024 patterns of m=16 over 256 KiB printable ASCII
    c3spec = rk.DnaSpec(seed=43, length=2**18, alphabet=ascii_alpha)
    c3 = rk.generate(c3spec)
    pats = []
    state = 43
    for j in range(512):
        draw, state = rk.splitmix64(state)
        x = draw % (len(c3) - 16 + 1)
        pats.append(c3[x:x + 16])
    for j in range(512):
        pats.append(rk.generate(rk.DnaSpec(seed=(43 ^ 0x5DEECE66D) + j, length=16,
                                           alphabet=ascii_alpha)))
    pats.append(b"a" * 15 + b"c")  # colliding pair inside the big set
    pats.append(b"a" * 14 + b"ba")
    addm("c3-256KiB-1026x16", c3, pats)
    (OUT / "multi_cases.json").write_text(json.dumps(multi))

    # ------------------------------------------------------------------ launch algebra
    launch = {"plan": [], "offset_of": []}
    for n, m, b, cap in [(1000, 7, 256, 65535), (100, 100, 32, 65535), (10_000_000, 7, 32, 65535),
                         (20_000, 1, 1, 10), (2**30, 16, 256, 65535), (2**34, 32, 1024, 65535),
                         (2**34, 32, 32, 65535)]:
        cfg = rk.plan_launch(n, m, b, cap)
        launch["plan"].append({"n": n, "m": m, "block": b, "cap": cap,
                               "grid": list(cfg.grid_dims), "total": cfg.total_threads})
    for (bx, by, bz), t, dims, b in [((0, 0, 0), 0, (4, 4, 1), 256), ((1, 2, 0), 3, (4, 4, 1), 256),
                                     ((0, 0, 1), 0, (4, 4, 2), 32), ((3, 2, 1), 31, (4, 3, 2), 32)]:
        x = rk.offset_of(rk.ThreadCoord((bx, by, bz), t), rk.LaunchConfig(dims, b))
        launch["offset_of"].append({"block_idx": [bx, by, bz], "thread": t, "grid": list(dims),
                                    "block": b, "offset": x})
    (OUT / "launch.json").write_text(json.dumps(launch))

    # ------------------------------------------------------------------ acceptance suite
    acceptance(rk, _scan)
    print("golden fixtures written to", OUT)


def _digest(values, dtype) -> str:
    return hashlib.sha1(np.asarray(values, dtype=dtype).tobytes()).hexdigest()[:16]


def acceptance(rk, _scan) -> None:
    """acceptance.json: the reference's own acceptance criteria 1, 4 and 5
    (/root/reference/pkg/tests/test_acceptance.py:49-85, :124-153, :156-182) recorded
    case by case.  The inputs are NOT stored: tests regenerate them from the same numpy
    seeds and draw sequence (tests/_golden.acceptance_cases), so only the reference's
    answers are kept -- per case (n, m, k, match count, collisions, sha1 of the int64
    offsets)."""
    acc = {}
    rng = np.random.default_rng(20240810)
    crit1 = []
    for case in range(10_008):
        k = (2, 4, 256)[case % 3]
        n = int(rng.integers(1, 4097))
        m = int(rng.integers(1, 65))
        text = rng.integers(0, k, size=n, dtype=np.uint8).tobytes()
        if m <= n and rng.random() < 0.5:
            x = int(rng.integers(0, n - m + 1))
            pattern = text[x: x + m]
        else:
            pattern = rng.integers(0, k, size=m, dtype=np.uint8).tobytes()
        st = rk.ScanStats()
        res = rk.search_sequential(text, pattern, stats=st)
        if case % 50 == 0:  # the reference's own equivalences, spot-checked here
            assert res == rk.search_naive(text, pattern)
            cfg = rk.plan_launch(n, m, 32) if m <= n else rk.LaunchConfig((1, 1, 1), 32)
            assert rk.search_parallel(text, pattern, cfg, 4) == res
        crit1.append([n, m, k, len(res.offsets), st.collisions, _digest(res.offsets, np.int64)])
    acc["criterion1"] = crit1

    filler = rk.generate(rk.DnaSpec(seed=11, length=5000))
    texts = [b"ac" + b"Xba" * 300, rk.plant(filler, b"ba", list(range(0, 4000, 13))),
             b"ba" * 64 + b"ac" + b"ba" * 64]
    crit4 = []
    for ti, text in enumerate(texts):
        for pattern in (b"ac", b"ba"):
            st = rk.ScanStats()
            res = rk.search_sequential(text, pattern, stats=st)
            multi = dict(rk.search_multi(text, rk.PatternSet([pattern])))
            assert multi[0] == res
            crit4.append({"text": ti, "pattern": pattern.decode(), "offsets": res.offsets,
                          "collisions": st.collisions, "hash_hits": st.hash_hits})
    acc["criterion4"] = crit4

    rng = np.random.default_rng(5150)
    crit5 = []
    for _ in range(1000):
        n = int(rng.integers(2, 4097))
        m = int(rng.integers(1, 65))
        if m >= n:
            m = n - 1 or 1
        text = rng.integers(0, 256, size=n, dtype=np.uint8).tobytes()
        h = _scan.window_hashes(_scan.as_u8(text), m, 0, n - m + 1)
        roll = [rk.hash_window(text, 0, m)]
        for x in range(n - m):
            roll.append(rk.roll(roll[-1], text[x], text[x + m], m))
        assert [int(v) for v in h] == roll
        crit5.append([n, m, _digest(h, np.uint64)])
    base = bytes(rng.integers(0, 256, size=80, dtype=np.uint8))
    acc["criterion5"] = crit5
    acc["criterion5_m65"] = {"base": enc(base), "h": str(rk.hash_window(base, 0, 65))}
    (OUT / "acceptance.json").write_text(json.dumps(acc, separators=(",", ":")))


if __name__ == "__main__":
    main()
