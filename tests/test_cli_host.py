"""CPU: the command line's host logic (mirrors pkg/tests/test_cli.py): span
grammar, config hash (equal to the reference's for the same fields), config
files, model subcommand rows, and configuration errors (exit code 2)."""

import csv
import io
import json
import os

import pytest

from paper_1006_3148_b200.cli import RunConfig, main, parse_span

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "perfmodel.json")))


def run(argv, capsys):
    code = main(argv)
    out = capsys.readouterr()
    return code, out.out, out.err


def rows(text):
    return list(csv.DictReader(io.StringIO(text)))


def test_parse_span_grammar():
    assert parse_span("1:4") == [1, 2, 3, 4]
    assert parse_span("0:8:2") == [0, 2, 4, 6, 8]
    assert parse_span("2,8,16") == [2, 8, 16]
    with pytest.raises(ValueError):
        parse_span("1:10:0")


def test_config_hash_equals_reference():
    h = GOLD["cli_config_hash"]
    assert RunConfig().config_hash() == h["default"]
    assert RunConfig(d_u=7).config_hash() == h["d_u=7"]
    assert RunConfig(nx=16, ny=16, nz=16, t=2, bx=16, by=8, bz=8,
                     mode="compressed").config_hash() == h["grid16_t2_compressed"]


def test_bad_configs_exit_2(tmp_path, capsys):
    code, _, err = run(["solve", "--grid", "16", "--block", "32,8,8"], capsys)
    assert code == 2 and "config error" in err
    cfg = tmp_path / "run.cfg"
    cfg.write_text("warp_factor = 9\n")
    assert run(["solve", "--config", str(cfg)], capsys)[0] == 2
    cfg.write_text("nx 16\n")
    assert run(["solve", "--config", str(cfg)], capsys)[0] == 2
    assert run(["dist", "--topo", "2,1,1", "--grid", "25", "--t", "2", "--block", "12,8,8"], capsys)[0] == 2
    assert run(["model", "--op", "baseline", "--machine", "/nonexistent/m.model"], capsys)[0] == 2


def test_model_rows(capsys):
    code, out, _ = run(["model", "--op", "baseline"], capsys)
    assert code == 0
    (r,) = rows(out)
    assert r["machine"] == "NVIDIA B200" and float(r["baseline_mlups"]) == GOLD["baseline_perf"] / 1e6
    code, out, _ = run(["model", "--op", "cycles", "--json"], capsys)
    got = {r["level"]: r for r in json.loads(out)}
    assert set(got) == {"smem", "L2", "HBM"}
    assert got["L2"]["cycles_max"] == GOLD["cache_cycle_model"]["L2"][1]
    code, out, _ = run(["model", "--op", "scalability", "--t-range", "0:400:100"], capsys)
    flags = [r["scales"] for r in rows(out)]
    assert flags[0] == "True" and flags[-1] == "False"
    code, out, _ = run(["model", "--op", "multihalo", "--L", "16,1024", "--h", "1,8"], capsys)
    got = {(int(r["L"]), int(r["h"])): float(r["multihalo"]) for r in rows(out)}
    assert got[(16, 8)] == pytest.approx(GOLD["multihalo_advantage"]["16,8"], rel=1e-12)
    assert got[(1024, 1)] == 1.0
