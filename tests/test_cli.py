"""CLI contract (reference cli.py: exit codes 0/1/2, MATCH/TOTAL listing)."""

import pytest

from paper_1810_01051_b200 import cli


def test_parse_size():
    assert cli.parse_size("10") == 10
    assert cli.parse_size("2KB") == 2048
    assert cli.parse_size("3MB") == 3 << 20
    assert cli.parse_size("1GB") == 1 << 30
    with pytest.raises(cli.CliError):
        cli.parse_size("x")
    with pytest.raises(cli.CliError):
        cli.parse_size("-5")


def test_errors_exit_2(tmp_path, capsys):
    f = tmp_path / "t.txt"
    f.write_bytes(b"abab")
    pf = tmp_path / "p.txt"
    pf.write_bytes(b"ab\n\nba\n")
    assert cli.main(["search", str(tmp_path / "missing"), "--pattern", "ab"]) == 2
    assert cli.main(["search", str(f)]) == 2
    assert cli.main(["search", str(f), "--pattern", "ab", "--pattern-file", str(pf)]) == 2
    assert cli.main(["search", str(f), "--pattern-file", str(pf)]) == 2  # blank line
    assert cli.main(["search", str(f), "--pattern", ""]) == 2
    assert cli.main(["bogus"]) == 2
    (tmp_path / "e.txt").write_bytes(b"")
    assert cli.main(["search", str(f), "--pattern-file", str(tmp_path / "e.txt")]) == 2


def test_naive_engine_listing(tmp_path, capsys):
    f = tmp_path / "t.txt"
    f.write_bytes(b"abab")
    assert cli.main(["search", str(f), "--pattern", "ab", "--engine", "naive"]) == 0
    assert capsys.readouterr().out.split("\n")[:3] == ["MATCH 0 0", "MATCH 0 2", "TOTAL 2"]
    assert cli.main(["search", str(f), "--pattern", "zz", "--engine", "naive"]) == 1


@pytest.mark.gpu
def test_gpu_engines_listing(tmp_path, capsys, gpu):
    f = tmp_path / "t.txt"
    f.write_bytes(b"abab")
    pf = tmp_path / "p.txt"
    pf.write_bytes(b"ab\nba\nab\nabc\n")
    for engine in ("seq", "par", "gpu"):
        assert cli.main(["search", str(f), "--pattern", "ab", "--engine", engine]) == 0
        assert capsys.readouterr().out.split("\n")[:3] == ["MATCH 0 0", "MATCH 0 2", "TOTAL 2"]
        assert cli.main(["search", str(f), "--pattern-file", str(pf), "--engine", engine]) == 0
        assert capsys.readouterr().out.strip().split("\n") == [
            "MATCH 0 0", "MATCH 1 1", "MATCH 0 2", "TOTAL 3"]
    assert cli.main(["verify", str(f), "--pattern-file", str(pf)]) == 0
    assert capsys.readouterr().out.startswith("PASS 3 pattern(s)")
    out = tmp_path / "g.txt"
    assert cli.main(["gen", "--size", "4KB", "--out", str(out)]) == 0
    assert out.stat().st_size == 4096
