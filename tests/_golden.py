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
