"""GPU tests of the C ABI's per-context state: the overflow protocol without a rescan
(rk_scan_fetch), stream ordering of the shared scratch across streams, and the pattern
cache's asynchronous upload.  Reference: _scan.py:53-68 (capacity, overflow -> rescan),
which the B200 path replaces by re-running only the ordered emission."""

import ctypes

import numpy as np
import pytest

import oracle
import paper_1810_01051_b200 as rk
from paper_1810_01051_b200 import _lib, _scan

pytestmark = pytest.mark.gpu


def _torch():
    import torch

    return torch


def test_dense_overflow_scans_once(gpu):
    """256 MiB of 'a' with 'aaaa' (C5): 2^28 - 3 matches overflow the first 65,536-offset
    buffer; the full list comes from a second EMIT, not a second scan: exactly one scan
    kernel and two emit kernels are launched."""
    torch = _torch()
    n = 1 << 28
    text = torch.full((n,), ord("a"), dtype=torch.uint8, device="cuda")
    ctx = _lib.context(0)
    before = ctx.launches
    st = rk.ScanStats()
    offs, k, coll, hits = _scan.scan_counts(text, b"aaaa", rk.hash_full(b"aaaa"), 0, n - 3)
    launches = ctx.launches - before
    assert launches == 3, launches  # scan + emit + re-emit
    assert k == n - 3 and coll == 0 and hits == n - 3
    assert offs.numel() == n - 3
    assert torch.equal(offs, torch.arange(n - 3, device="cuda", dtype=torch.int64))
    r = rk.search_sequential(text[: 1 << 20], b"aaaa", stats=st)
    assert r.offsets == list(range((1 << 20) - 3))


def test_fetch_without_device_scan_is_einval(gpu):
    torch = _torch()
    ctx = _lib.context(0)
    L = _lib.lib()
    host = np.frombuffer(b"abcabcabc" * 100, dtype=np.uint8)
    out = np.empty(16, dtype=np.int64)
    mt, co, hh = _lib.u64ref(), _lib.u64ref(), _lib.u64ref()
    pat = np.frombuffer(b"abc", dtype=np.uint8)
    with ctx.lock:
        _lib.check(L.rk_scan_host(ctx.handle, host.ctypes.data, host.size, pat.ctypes.data, 3,
                                  rk.hash_full(b"abc"), 0, host.size - 2, out.ctypes.data, 16,
                                  ctypes.byref(mt), ctypes.byref(co), ctypes.byref(hh)))
        d = torch.empty(300, dtype=torch.int64, device="cuda")
        with pytest.raises(ValueError):
            _lib.check(L.rk_scan_fetch(ctx.handle, d.data_ptr(), 300, _scan._stream(0)))


def test_fetch_reemits_same_list(gpu):
    """rk_scan with a small cap, then rk_scan_fetch: the same ordered list as a scan with
    room for all of them, for a sparse and a dense pattern."""
    torch = _torch()
    spec = rk.DnaSpec(7, 1 << 22, b"ab")
    text = rk.generate_tensor(spec, device="cuda")
    host = text.cpu().numpy()
    L = _lib.lib()
    ctx = _lib.context(0)
    s = _scan._stream(0)
    for pat in (b"abba", b"aaaaaaaaaaaa", b"ab"):
        p = np.frombuffer(pat, dtype=np.uint8)
        exp, ecoll = oracle.c_scan(host, p)
        mt, co, hh = _lib.u64ref(), _lib.u64ref(), _lib.u64ref()
        small = torch.empty(5, dtype=torch.int64, device="cuda")
        with ctx.lock:
            _lib.check(L.rk_scan(ctx.handle, text.data_ptr(), text.numel(), p.ctypes.data,
                                 len(pat), rk.hash_full(pat), 0, text.numel() - len(pat) + 1,
                                 small.data_ptr(), 5, ctypes.byref(mt), ctypes.byref(co),
                                 ctypes.byref(hh), s))
            k = int(mt.value)
            assert k == len(exp) and int(co.value) == ecoll
            big = torch.empty(k, dtype=torch.int64, device="cuda")
            _lib.check(L.rk_scan_fetch(ctx.handle, big.data_ptr(), k, s))
            # a second fetch of the same scan is allowed too
            again = torch.empty(k, dtype=torch.int64, device="cuda")
            _lib.check(L.rk_scan_fetch(ctx.handle, again.data_ptr(), k, s))
        assert big.cpu().numpy().tolist() == exp.tolist()
        assert torch.equal(big, again)
        assert small.cpu().numpy().tolist() == exp[:5].tolist()


def test_scans_on_alternating_streams(gpu):
    """Async scans of one context issued on two streams in turn with no host sync in
    between (the scratch -- per-tile results, counter sets, pattern slots -- is ordered
    across each switch): every offset list and counter set is exact."""
    torch = _torch()
    spec = rk.DnaSpec(3, 1 << 24, b"ACGT")
    text = rk.generate_tensor(spec, device="cuda")
    host = text.cpu().numpy()
    n = text.numel()
    L = _lib.lib()
    ctx = _lib.context(0)
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    pats = [host[x : x + m].tobytes() for x, m in ((5, 6), (1000, 9), (77, 4), (4096, 13),
                                                    (12345, 70), (999, 5), (31, 8), (8, 33))]
    # more distinct patterns than the 64-slot pattern cache: slots are re-uploaded while
    # the other stream may still be reading them
    pats += [host[x : x + 10].tobytes() for x in range(100, 100 + 70 * 97, 97)]
    cap = 1 << 16
    outs = torch.empty((len(pats), cap), dtype=torch.int64, device="cuda")
    cnts = torch.zeros((len(pats), 3), dtype=torch.int64, device="cuda")
    torch.cuda.synchronize()
    keep = []
    with ctx.lock:
        for i, pat in enumerate(pats):
            p = np.frombuffer(pat, dtype=np.uint8)
            keep.append(p)
            _lib.check(L.rk_scan_async(ctx.handle, text.data_ptr(), n, p.ctypes.data, len(pat),
                                       rk.hash_full(pat), 0, n - len(pat) + 1,
                                       outs[i].data_ptr(), cap, 0, cnts[i].data_ptr(),
                                       streams[i % 2].cuda_stream))
    torch.cuda.synchronize()
    c = cnts.cpu().numpy()
    o = outs.cpu().numpy()
    for i, pat in enumerate(pats):
        exp, ecoll = oracle.c_scan(host, np.frombuffer(pat, dtype=np.uint8))
        k = int(c[i, 0])
        assert k == len(exp) and int(c[i, 2]) == ecoll and int(c[i, 1]) == k + ecoll, i
        assert o[i, : min(k, cap)].tolist() == exp[:cap].tolist(), i


def test_concurrent_callers_get_their_own_contexts(gpu):
    """The reference runs range scans concurrently on a thread pool
    (parallel.py:111-121, :162-167).  Concurrent Python callers here each hold their own
    context (_lib.acquire: the primary one if free, else a pooled spare), so host-text
    and device-text scans from 6 threads run side by side and all stay exact."""
    import threading

    import oracle

    torch = _torch()
    rng = np.random.default_rng(31)
    texts = [rng.integers(0, 4, (1 << 20) + 977 * i, dtype=np.uint8) for i in range(6)]
    pats = [t[4000:4000 + m].tobytes() for t, m in zip(texts, (4, 8, 13, 32, 64, 200))]
    expect = [oracle.c_scan(t, np.frombuffer(p, np.uint8)) for t, p in zip(texts, pats)]
    errors = []

    def work(i):
        try:
            torch.cuda.set_device(0)
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                for rep in range(20):
                    src = texts[i] if rep % 2 else torch.from_numpy(texts[i]).cuda()
                    st = rk.ScanStats()
                    r = rk.search_sequential(src, pats[i], stats=st)
                    assert r.offsets == expect[i][0].tolist() and st.collisions == expect[i][1]
        except Exception as e:  # noqa: BLE001
            errors.append((i, repr(e)))

    th = [threading.Thread(target=work, args=(i,)) for i in range(6)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errors, errors


def test_dense_tiles_queued_with_caps(gpu):
    """Dense stretches (all 'a') inside a sparse text: the emit queues the dense tiles for
    its balanced phase and expands the sparse ones in place; the ordered list -- also cut
    at caps inside dense and sparse tiles, and re-emitted by rk_scan_fetch -- equals the
    oracle's."""
    torch = _torch()
    rng = np.random.default_rng(11)
    host = rng.integers(0, 4, 24 << 20, dtype=np.uint8) + ord("a")
    for x, ln in ((1 << 20, 3 << 20), (9 << 20, 1 << 20), ((20 << 20) + 77, 777_777)):
        host[x:x + ln] = ord("a")
    text = torch.from_numpy(host).cuda()
    L = _lib.lib()
    ctx = _lib.context(0)
    s = _scan._stream(0)
    for pat in (b"aa", b"aaaa", b"ab"):
        p = np.frombuffer(pat, dtype=np.uint8)
        exp, ecoll = oracle.c_scan(host, p)
        for cap in (len(exp), len(exp) - 1, (1 << 20) + 5, 1000):
            out = torch.full((cap,), -1, dtype=torch.int64, device="cuda")
            mt, co, hh = _lib.u64ref(), _lib.u64ref(), _lib.u64ref()
            with ctx.lock:
                _lib.check(L.rk_scan(ctx.handle, text.data_ptr(), text.numel(), p.ctypes.data,
                                     len(pat), rk.hash_full(pat), 0, text.numel() - len(pat) + 1,
                                     out.data_ptr(), cap, ctypes.byref(mt), ctypes.byref(co),
                                     ctypes.byref(hh), s))
            assert int(mt.value) == len(exp) and int(co.value) == ecoll
            assert np.array_equal(out.cpu().numpy(), exp[:cap])
        with ctx.lock:
            full = torch.empty(len(exp), dtype=torch.int64, device="cuda")
            _lib.check(L.rk_scan_fetch(ctx.handle, full.data_ptr(), len(exp), s))
        assert np.array_equal(full.cpu().numpy(), exp)


def test_emit_queue_fuzz(gpu):
    """Randomised texts of dense stretches (one letter, or two letters alternating) inside
    sparse random text, m = 1..12, scanned through the C ABI with random caps and then
    re-emitted in full (rk_scan_fetch): the dense tiles go through the emit's queue, the
    rest is expanded in place, and every list, cut and count equals the oracle's."""
    torch = _torch()
    rng = np.random.default_rng(4242)
    L = _lib.lib()
    ctx = _lib.context(0)
    s = _scan._stream(0)
    for case in range(40):
        n = int(rng.integers(1 << 16, 6 << 20))
        host = rng.integers(ord("a"), ord("e"), n, dtype=np.uint8)
        for _ in range(int(rng.integers(1, 6))):
            ln = int(rng.integers(1, 1 << 20))
            x = int(rng.integers(0, n))
            seg = host[x:x + ln]
            if rng.random() < 0.5:
                seg[:] = ord("a")
            else:
                seg[0::2] = ord("a")
                seg[1::2] = ord("b")
        m = int(rng.integers(1, 13))
        pat = (b"a" * m) if rng.random() < 0.5 else bytes((b"ab" * 8)[:m])
        p = np.frombuffer(pat, dtype=np.uint8)
        exp, ecoll = oracle.c_scan(host, p, workers=8)
        text = torch.from_numpy(host).cuda()
        cap = int(rng.integers(0, len(exp) + 2)) if len(exp) else 0
        out = torch.full((max(cap, 1),), -1, dtype=torch.int64, device="cuda")
        mt, co, hh = _lib.u64ref(), _lib.u64ref(), _lib.u64ref()
        with ctx.lock:
            _lib.check(L.rk_scan(ctx.handle, text.data_ptr(), n, p.ctypes.data, m,
                                 rk.hash_full(pat), 0, n - m + 1, out.data_ptr(), cap,
                                 ctypes.byref(mt), ctypes.byref(co), ctypes.byref(hh), s))
            k = int(mt.value)
            assert k == len(exp) and int(co.value) == ecoll and int(hh.value) == k + ecoll, case
            full = torch.empty(max(k, 1), dtype=torch.int64, device="cuda")
            if k:
                _lib.check(L.rk_scan_fetch(ctx.handle, full.data_ptr(), k, s))
        assert np.array_equal(out[:min(cap, k)].cpu().numpy(), exp[:cap]), (case, n, m, cap)
        assert np.array_equal(full[:k].cpu().numpy(), exp), (case, n, m)
