"""Loader for the golden fixtures written by tests/golden/make_golden.py (from the
reference itself)."""

from __future__ import annotations

import base64
import json
import zlib
from functools import lru_cache
from pathlib import Path

GOLDEN = Path(__file__).resolve().parent / "golden"


def dec(s: str) -> bytes:
    return zlib.decompress(base64.b64decode(s))


@lru_cache(maxsize=None)
def load(name: str):
    return json.loads((GOLDEN / name).read_text())


def scan_cases():
    out = []
    for c in load("scan_cases.json"):
        d = dict(c)
        d["text"] = dec(c["text"])
        d["pattern"] = dec(c["pattern"])
        out.append(d)
    return out


def multi_cases():
    out = []
    for c in load("multi_cases.json"):
        d = dict(c)
        d["text"] = dec(c["text"])
        d["patterns"] = [dec(p) for p in c["patterns"]]
        d["deduped"] = [dec(p) for p in c["deduped"]]
        out.append(d)
    return out


def corpus():
    return load("corpus.json")


def hash_kat():
    return load("hash_kat.json")


def launch():
    return load("launch.json")


ASCII = bytes(range(32, 127))


def acceptance():
    return load("acceptance.json")


def criterion1_cases():
    """The 10,008 cases of the reference's criterion 1
    (/root/reference/pkg/tests/test_acceptance.py:49-85), regenerated from the same seed
    and draw sequence, each with the reference's recorded answer:
    yields (case, text, pattern, workers, block_dim, expected) with expected =
    [n, m, k, matches, collisions, sha1-16 of the int64 offsets]."""
    import numpy as np

    rng = np.random.default_rng(20240810)
    workers_grid, block_grid = (1, 2, 4, 8), (32, 256, 1024)
    for case, exp in enumerate(acceptance()["criterion1"]):
        k = (2, 4, 256)[case % 3]
        n = int(rng.integers(1, 4097))
        m = int(rng.integers(1, 65))
        text = rng.integers(0, k, size=n, dtype=np.uint8).tobytes()
        if m <= n and rng.random() < 0.5:
            x = int(rng.integers(0, n - m + 1))
            pattern = text[x: x + m]
        else:
            pattern = rng.integers(0, k, size=m, dtype=np.uint8).tobytes()
        assert exp[:3] == [n, m, k], (case, exp[:3], (n, m, k))  # draw sequence in step
        yield (case, text, pattern, workers_grid[case % 4], block_grid[(case // 4) % 3], exp)


def criterion5_texts():
    """The 1,000 texts of criterion 5 (test_acceptance.py:156-182): yields (text, m,
    sha1-16 of the reference's uint64 window hashes)."""
    import numpy as np

    rng = np.random.default_rng(5150)
    for exp in acceptance()["criterion5"]:
        n = int(rng.integers(2, 4097))
        m = int(rng.integers(1, 65))
        if m >= n:
            m = n - 1 or 1
        text = rng.integers(0, 256, size=n, dtype=np.uint8).tobytes()
        assert exp[:2] == [n, m]
        yield text, m, exp[2]


def digest(values, dtype) -> str:
    import hashlib

    import numpy as np

    return hashlib.sha1(np.asarray(values, dtype=dtype).tobytes()).hexdigest()[:16]
