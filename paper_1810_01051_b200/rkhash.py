"""Shift-add window hash -- same definition as the reference (rkmatch.rkhash).

h(b_0 .. b_{m-1}) = sum b_i * 2^(m-1-i) mod 2^64 : base 2, the word width as the
modulus, raw byte values (/root/reference/pkg/src/rkmatch/rkhash.py:1-28).  Only the
last 64 bytes can contribute (earlier coefficients are 0 mod 2^64), which this host
implementation uses directly; the device kernels use the exact 32-bit roll derived from
``roll`` (rkhash.py:48-60).
"""

from __future__ import annotations

MASK64 = (1 << 64) - 1

HashValue = int


def _bytes(data) -> bytes:
    if isinstance(data, bytes):
        return data
    try:
        import torch

        if isinstance(data, torch.Tensor):
            return data.detach().to("cpu").contiguous().numpy().tobytes()
    except ImportError:  # pragma: no cover
        pass
    return bytes(data)


def hash_full(data) -> HashValue:
    """Hash an entire byte string; the empty string hashes to 0 (rkhash.py:21-28)."""
    b = _bytes(data)
    h = 0
    for x in b[-64:]:
        h = (h << 1) + x
    return h & MASK64


def hash_window(text, offset: int, m: int) -> HashValue:
    """Hash of text[offset:offset+m]; ValueError on m < 1 or out of range (rkhash.py:31-45)."""
    if m < 1:
        raise ValueError("window length must be >= 1")
    if offset < 0 or offset + m > len(text):
        raise ValueError(
            f"window [{offset}, {offset + m}) out of range for text of length {len(text)}"
        )
    return hash_full(_bytes(text[offset : offset + m]))


def roll(prev: HashValue, outgoing: int, incoming: int, m: int) -> HashValue:
    """Slide the hash of text[x:x+m] to text[x+1:x+m+1] (rkhash.py:48-60)."""
    if m < 1:
        raise ValueError("window length must be >= 1")
    top = (outgoing << (m - 1)) & MASK64
    return (((prev - top) << 1) + incoming) & MASK64
