"""Synthetic corpora -- bit-identical to rkmatch.datagen, generated on the B200.

The reference stream is counter-based (/root/reference/pkg/src/rkmatch/datagen.py:1-77):
byte i of a (seed, length, alphabet) corpus is alphabet[z_{i+1} mod k] with
z_s = mix(seed + s * GOLDEN), so any slice of a 16 GiB corpus can be produced directly
in HBM, shard-local, by ``rk_generate``.  ``generate`` returns bytes
like the reference; ``generate_tensor`` leaves the corpus on the device.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib
from .rkhash import MASK64

_GOLDEN = 0x9E3779B97F4A7C15
_MIX1 = 0xBF58476D1CE4E5B9
_MIX2 = 0x94D049BB133111EB

DNA_ALPHABET = b"ACGT"
ASCII_PRINTABLE = bytes(range(32, 127))


def splitmix64(state: int) -> tuple[int, int]:
    """One splitmix64 step; returns (output, next state) (datagen.py:28-34)."""
    state = (state + _GOLDEN) & MASK64
    z = state
    z = ((z ^ (z >> 30)) * _MIX1) & MASK64
    z = ((z ^ (z >> 27)) * _MIX2) & MASK64
    return z ^ (z >> 31), state


def splitmix64_stream(seed: int, count: int, skip: int = 0) -> np.ndarray:
    """Outputs for steps skip+1 .. skip+count (datagen.py:37-48)."""
    if count < 0:
        raise ValueError("count must be >= 0")
    steps = np.arange(skip + 1, skip + count + 1, dtype=np.uint64)
    z = np.uint64(seed & MASK64) + np.uint64(_GOLDEN) * steps
    z = (z ^ (z >> np.uint64(30))) * np.uint64(_MIX1)
    z = (z ^ (z >> np.uint64(27))) * np.uint64(_MIX2)
    return z ^ (z >> np.uint64(31))


@dataclass(frozen=True)
class DnaSpec:
    """Seed, length and alphabet of one reproducible corpus (datagen.py:51-65)."""

    seed: int
    length: int
    alphabet: bytes = DNA_ALPHABET

    def __post_init__(self):
        if self.length < 0:
            raise ValueError("length must be >= 0")
        if not self.alphabet:
            raise ValueError("alphabet must not be empty")
        if len(set(self.alphabet)) != len(self.alphabet):
            raise ValueError("alphabet symbols must be distinct")


def generate_into(out, spec: DnaSpec, skip: int = 0, stream=None) -> None:
    """Write corpus bytes [skip, skip + out.numel()) of ``spec`` into a CUDA uint8 tensor."""
    import torch

    dev = out.device.index if out.device.index is not None else torch.cuda.current_device()
    alpha = np.frombuffer(spec.alphabet, dtype=np.uint8)
    s = stream if stream is not None else torch.cuda.current_stream(dev).cuda_stream
    with _lib.acquire(dev) as ctx:
        _lib.check(_lib.lib().rk_generate(ctx.handle, out.data_ptr(), int(out.numel()),
                                          spec.seed & MASK64, skip, alpha.ctypes.data,
                                          len(spec.alphabet), s))


def generate_tensor(spec: DnaSpec, device=None, skip: int = 0, count: int | None = None):
    """Corpus slice [skip, skip + count) as a CUDA uint8 tensor."""
    import torch

    if device is None:
        device = f"cuda:{_lib.default_device()}"
    count = spec.length - skip if count is None else count
    out = torch.empty(count, dtype=torch.uint8, device=device)
    if count:
        generate_into(out, spec, skip)
    return out


def generate(spec: DnaSpec) -> bytes:
    """Deterministic corpus of exactly spec.length alphabet bytes (datagen.py:68-77)."""
    if spec.length == 0:
        return b""
    return generate_tensor(spec).cpu().numpy().tobytes()


def plant(text, pattern, offsets) -> bytes:
    """Copy of ``text`` with ``pattern`` spliced in at each offset (datagen.py:80-102)."""
    text = text if isinstance(text, bytes) else bytes(text)
    pattern = pattern if isinstance(pattern, bytes) else bytes(pattern)
    m = len(pattern)
    if m == 0:
        raise ValueError("empty pattern")
    ordered = sorted(offsets)
    for x in ordered:
        if x < 0 or x + m > len(text):
            raise ValueError(f"offset {x} out of range for pattern of length {m}")
    for a, b in zip(ordered, ordered[1:]):
        if b - a < m:
            raise ValueError(f"offsets {a} and {b} overlap for pattern length {m}")
    buf = bytearray(text)
    for x in ordered:
        buf[x : x + m] = pattern
    return bytes(buf)


def make_pattern(text, spec: DnaSpec, m: int, source: str) -> bytes:
    """The benchmark pattern of rkmatch.bench._make_pattern (bench.py:106-119)."""
    if m < 1:
        raise ValueError("pattern length must be >= 1")
    n = len(text) if not hasattr(text, "numel") else int(text.numel())
    if m > n:
        raise ValueError(f"pattern length {m} exceeds corpus length {n}")
    if source == "sampled":
        draw, _ = splitmix64(spec.seed ^ 0xA5A5A5A5A5A5A5A5)
        x = draw % (n - m + 1)
        piece = text[x : x + m]
        if hasattr(piece, "cpu"):
            return piece.cpu().numpy().tobytes()
        return bytes(piece)
    if source == "generated":
        return generate(DnaSpec(seed=spec.seed ^ 0x5DEECE66D, length=m, alphabet=spec.alphabet))
    raise ValueError(f"unknown pattern source {source!r}")

