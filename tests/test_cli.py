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


def test_bench_validation_and_formats(capsys):
    from paper_1810_01051_b200 import bench

    with pytest.raises(ValueError):
        bench.sweep("nope", [1])
    with pytest.raises(ValueError):
        bench.sweep("workers", [])
    with pytest.raises(ValueError):
        bench.sweep("workers", [1], bench.SweepConfig(reps=2))
    with pytest.raises(ValueError):
        bench.speedup(0, 1)
    assert bench.speedup(6.0, 2.0) == 3.0
    rep = bench.BenchReport("pattern_length", [bench.BenchRow(25, 2.0, 1.0, 2.0)], {},
                            [bench.DeviceRow(25, 0.5, 40.0, 3)])
    assert bench.format_csv(rep) == "axis_value,t_seq_ms,t_par_ms,speedup\n25,2.0,1.0,2.0\n"
    table = bench.format_table(rep).split("\n")
    assert table[0].split() == ["pattern_length", "t_seq_ms", "t_par_ms", "speedup",
                                "t_dev_ms", "dev_GB/s"]
    assert table[2].split()[:4] == ["25", "2.000", "1.000", "2.0000"]
    payload = bench.report_payload(rep)
    assert payload["rows"] == [{"axis_value": 25, "t_seq_ms": 2.0, "t_par_ms": 1.0, "speedup": 2.0}]
    assert payload["device_rows"][0]["gbps"] == 40.0
    assert cli.main(["bench", "--axis", "bogus", "--values", "1"]) == 2
    assert cli.main(["bench", "--axis", "workers", "--values", ","]) == 2
    assert cli.main(["bench", "--axis", "workers", "--values", "x"]) == 2


@pytest.mark.gpu
def test_bench_sweep_gpu(tmp_path, capsys, gpu):
    import json

    from paper_1810_01051_b200 import bench

    cfg = bench.SweepConfig(corpus=bench.DnaSpec(42, 1 << 20), pattern_length=7)
    rep = bench.sweep("pattern_length", [5, 25], cfg)
    assert [r.axis_value for r in rep.rows] == [5, 25]
    assert all(r.speedup == r.t_seq_ms / r.t_par_ms for r in rep.rows)
    assert [r.axis_value for r in rep.device_rows] == [5, 25]
    assert all(r.matches >= 1 and r.t_dev_ms > 0 for r in rep.device_rows)
    base = tmp_path / "rep"
    assert cli.main(["bench", "--axis", "file_size", "--values", "300KB,1MB", "--size", "1MB",
                     "--out", str(base), "--format", "json"]) == 0
    data = json.loads((tmp_path / "rep.json").read_text())
    assert [r["axis_value"] for r in data["rows"]] == [300 << 10, 1 << 20]
    assert (tmp_path / "rep.csv").read_text().startswith("axis_value,t_seq_ms,t_par_ms,speedup\n")


def test_bench_reference_arm_line():
    """bench.py --impl reference: one JSON line with the contract's keys, same config as
    the GPU arm, the reference algorithm timed on the host cores (no GPU needed)."""
    import json
    import subprocess
    import sys
    from pathlib import Path

    root = Path(__file__).resolve().parent.parent
    r = subprocess.run([sys.executable, str(root / "bench.py"), "--impl", "reference",
                        "--steps", "1", "--warmup", "0", "--sweep", "32,64",
                        "--ref-seconds", "0.5"], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["unit"] == "GB/s" and line["value"] > 0
    for k in ("metric", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "dtype", "config", "cpu_baseline", "e2e"):
        assert k in line, k
    assert line["config"]["sweep"] == [32, 64]
    assert line["cpu_baseline"]["kind"] == "port" and line["cpu_baseline"]["value"] == line["value"]
    assert line["e2e"]["h2d_bytes_per_step"] == 0
