"""The reference's own acceptance criteria 1, 4 and 5
(/root/reference/pkg/tests/test_acceptance.py:49-85, :124-153, :156-182) run through the
B200 path.  Inputs are regenerated from the reference's seeds (tests/_golden.py); the
expected answers were recorded from the reference itself (tests/golden/make_golden.py)."""

import numpy as np
import pytest

import paper_1810_01051_b200 as rk
from paper_1810_01051_b200 import _scan

pytestmark = pytest.mark.gpu


def test_criterion1_all_10008_cases(gpu, golden):
    """naive == sequential == parallel for every case, worker count and block size: here
    sequential and parallel run on the GPU (host bytes in, rk_scan_host) and must equal
    the reference's recorded offsets and collision counts for all 10,008 cases."""
    checked = 0
    for case, text, pattern, workers, block, exp in golden.criterion1_cases():
        n, m = len(text), len(pattern)
        st = rk.ScanStats()
        r = rk.search_sequential(text, pattern, stats=st)
        assert (len(r.offsets), st.collisions, golden.digest(r.offsets, np.int64)) == \
            tuple(exp[3:]), case
        cfg = rk.plan_launch(n, m, block) if m <= n else rk.LaunchConfig((1, 1, 1), block)
        stp = rk.ScanStats()
        assert rk.search_parallel(text, pattern, cfg, workers, stats=stp) == r, case
        assert stp.collisions == st.collisions and stp.hash_hits == st.hash_hits, case
        checked += 1
    assert checked == 10_008


def test_criterion1_device_tensors(gpu, golden):
    """Every 7th criterion-1 case again with the text already in HBM (rk_scan on the
    current stream, CUDA offsets)."""
    import torch

    for case, text, pattern, _w, _b, exp in golden.criterion1_cases():
        if case % 7:
            continue
        t = torch.frombuffer(bytearray(text), dtype=torch.uint8).cuda()
        st = rk.ScanStats()
        r = rk.search_sequential(t, pattern, stats=st)
        assert (len(r.offsets), st.collisions, golden.digest(r.offsets, np.int64)) == \
            tuple(exp[3:]), case


def test_criterion4_collision_soundness(gpu, golden):
    filler = rk.generate(rk.DnaSpec(seed=11, length=5000))
    texts = [b"ac" + b"Xba" * 300, rk.plant(filler, b"ba", list(range(0, 4000, 13))),
             b"ba" * 64 + b"ac" + b"ba" * 64]
    total = 0
    for c in golden.acceptance()["criterion4"]:
        text, pattern = texts[c["text"]], c["pattern"].encode()
        expected = rk.search_naive(text, pattern)
        assert expected.offsets == c["offsets"]
        seq = rk.ScanStats()
        assert rk.search_sequential(text, pattern, stats=seq) == expected
        par = rk.ScanStats()
        cfg = rk.plan_launch(len(text), len(pattern), 32)
        assert rk.search_parallel(text, pattern, cfg, 4, stats=par) == expected
        assert seq.collisions == par.collisions == c["collisions"]
        assert seq.hash_hits == c["hash_hits"]
        assert dict(rk.search_multi(text, rk.PatternSet([pattern])))[0] == expected
        total += seq.collisions
    assert total > 0


def test_criterion5_window_hashes(gpu, golden):
    """The device window hashes (rk_window_hashes) of all 1,000 texts equal the
    reference's (which its rolling oracle was checked against)."""
    import torch

    for text, m, dig in golden.criterion5_texts():
        t = torch.frombuffer(bytearray(text), dtype=torch.uint8).cuda()
        h = _scan.window_hashes(t, m, 0, len(text) - m + 1)
        assert golden.digest(h.cpu().numpy(), np.uint64) == dig
