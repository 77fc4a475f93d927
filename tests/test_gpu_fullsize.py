"""Full-size GPU properties (BASELINE.json configs at their real sizes).

The oracle cannot scan 1-16 GiB in test time, so these use size-independent properties:
exact agreement with the oracle on prefixes and random slices, byte-verification of
every reported offset on the device, planted copies across tile/chunk/shard edges, the
analytic answer for all-'a', and counter identities."""

import numpy as np
import pytest

import oracle
import paper_1810_01051_b200 as rk
from paper_1810_01051_b200 import _scan
from tests import _golden as G

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

GiB = 1 << 30


def _verify_on_device(torch, t, offs, pat):
    """Every reported offset byte-equals the pattern; offsets strictly ascending."""
    m = len(pat)
    if offs.numel() == 0:
        return
    assert bool((offs[1:] > offs[:-1]).all())
    idx = offs.view(-1, 1) + torch.arange(m, device=t.device).view(1, -1)
    win = t[idx]
    p = torch.frombuffer(bytearray(pat), dtype=torch.uint8).to(t.device)
    assert bool((win == p.view(1, -1)).all())


def _slices_agree(text_host_fn, offs_host, pat, n, seed, samples=4, window=1 << 16):
    """rkmatch.bench._verify_subsampled (bench.py:122-147) with the oracle."""
    m = len(pat)
    state = seed
    for _ in range(samples):
        draw, state = oracle.splitmix64(state)
        a = draw % (n - window + 1)
        b = a + window
        piece = text_host_fn(a, b)
        eo, _ = oracle.c_scan(piece, np.frombuffer(pat, dtype=np.uint8))
        expect = (eo + a).tolist()
        lo = np.searchsorted(offs_host, a)
        hi = np.searchsorted(offs_host, b - m, side="right")
        assert offs_host[lo:hi].tolist() == expect, (a, b)


@pytest.mark.parametrize("m", [4, 5, 8, 12, 16, 20, 25, 32, 64, 128, 256, 512, 1024])
def test_c2_1gib_ascii(gpu, m):
    import torch

    spec = rk.DnaSpec(42, GiB, G.ASCII)
    t = rk.generate_tensor(spec)
    pat = rk.datagen.make_pattern(t, spec, m, "sampled")
    # plant copies straddling 16 KiB tile and 64 MiB staging boundaries
    plants = [k * (1 << 14) - 7 for k in (1, 2, 1000)] + [(64 << 20) - m // 2, GiB - m]
    p = torch.frombuffer(bytearray(pat), dtype=torch.uint8).cuda()
    for x in plants:
        t[x : x + m] = p
    hx = rk.hash_full(pat)
    offs, k, coll, hits = _scan.scan_counts(t, pat, hx, 0, GiB - m + 1)
    assert hits == k + coll
    _verify_on_device(torch, t, offs, pat)
    oh = offs.cpu().numpy()
    for x in plants:
        assert x in set(oh.tolist())
    # exact equality with the oracle on a 32 MiB prefix (counts collisions too)
    pre = 32 << 20
    host_pre = t[:pre].cpu().numpy()
    eo, ec = oracle.c_scan(host_pre, np.frombuffer(pat, dtype=np.uint8),
                           workers=oracle.cpu_threads())
    po, _, pc, _ = _scan.scan_counts(t[:pre], pat, hx, 0, pre - m + 1)
    assert po.cpu().numpy().tolist() == eo.tolist() and pc == ec
    _slices_agree(lambda a, b: t[a:b].cpu().numpy(), oh, pat, GiB, 42)


def test_c5_all_a_256mib(gpu):
    import torch

    n = 1 << 28
    t = torch.full((n,), 97, dtype=torch.uint8, device="cuda")
    offs, k, coll, hits = _scan.scan_counts(t, b"aaaa", rk.hash_full(b"aaaa"), 0, n - 3)
    assert k == n - 3 and coll == 0 and hits == n - 3
    assert torch.equal(offs, torch.arange(n - 3, device="cuda"))


def test_c4_dna_4gib_planted(gpu):
    import torch

    n = 4 * GiB
    spec = rk.DnaSpec(42, n)
    t = rk.generate_tensor(spec)
    pat = rk.datagen.make_pattern(t, spec, 32, "sampled")
    p = torch.frombuffer(bytearray(pat), dtype=torch.uint8).cuda()
    plants = [g * (n // 8) - 16 for g in range(1, 8)] + [(1 << 32) - 40]
    for x in plants:
        t[x : x + 32] = p
    offs, k, coll, hits = _scan.scan_counts(t, pat, rk.hash_full(pat), 0, n - 31)
    _verify_on_device(torch, t, offs, pat)
    got = set(offs.cpu().numpy().tolist())
    for x in plants:
        assert x in got
    assert coll == 0
    # 64-bit offsets beyond 2^32
    assert max(got) > (1 << 31)


def test_host_e2e_1gib_pinned(gpu):
    import torch

    spec = rk.DnaSpec(42, GiB, G.ASCII)
    t = rk.generate_tensor(spec)
    host = t.cpu().pin_memory()
    pat = rk.datagen.make_pattern(t, spec, 8, "sampled")
    st = rk.ScanStats()
    r = rk.search_sequential(host, pat, stats=st)
    dev_offs, k, coll, hits = _scan.scan_counts(t, pat, rk.hash_full(pat), 0, GiB - 7)
    assert r.offsets == dev_offs.cpu().numpy().tolist()
    assert st.collisions == coll and st.hash_hits == hits
