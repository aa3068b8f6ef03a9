"""GPU: the command line end to end (mirrors pkg/tests/test_cli.py): solve
with --verify (bit-exact against plain sweeps on the device), config files
and overrides, snapshot determinism and replay from an output row, sweep
rows, bench rows, and the in-process distributed run with --verify."""

import csv
import io

import pytest

pytestmark = pytest.mark.gpu

from paper_1006_3148_b200.cli import RunConfig, main  # noqa: E402


def run(argv, capsys):
    code = main(argv)
    out = capsys.readouterr()
    return code, out.out, out.err


def rows(text):
    return list(csv.DictReader(io.StringIO(text)))


@pytest.mark.parametrize("argv", [
    ["solve", "--grid", "16", "--t", "2", "--block", "16,8,8", "--passes", "2", "--verify"],
    ["solve", "--grid", "60", "--t", "3", "--T", "1", "--passes", "2", "--block", "60,20,20", "--verify"],
    ["solve", "--grid", "40", "--n", "2", "--t", "4", "--passes", "3", "--block", "40,8,8", "--verify"],
    ["solve", "--grid", "24", "--t", "3", "--mode", "compressed", "--block", "24,8,8", "--passes", "4",
     "--verify"],
])
def test_solve_verify_bitwise(argv, capsys):
    code, out, _ = run(argv, capsys)
    assert code == 0
    (r,) = rows(out)
    assert r["verified"] == "bitwise match" and float(r["mlups"]) > 0


def test_config_file_and_overrides(tmp_path, capsys):
    cfg = tmp_path / "run.cfg"
    cfg.write_text("nx = 16\nny = 16\nnz = 16\nt = 2\nbx = 16\nby = 8\nbz = 8\npasses = 2\n")
    code, out, _ = run(["solve", "--config", str(cfg), "--verify"], capsys)
    (r,) = rows(out)
    assert code == 0 and r["t"] == "2" and r["nx"] == "16"
    code, out, _ = run(["solve", "--config", str(cfg), "--t", "1", "--verify"], capsys)
    (r,) = rows(out)
    assert code == 0 and r["t"] == "1"


def test_snapshot_determinism_and_replay(tmp_path, capsys):
    outs = []
    for name in ("a.grid", "b.grid"):
        code, out, _ = run(["solve", "--grid", "16", "--n", "2", "--t", "2", "--mode", "compressed",
                            "--block", "16,8,8", "--passes", "2", "--out", str(tmp_path / name)], capsys)
        assert code == 0
        (r,) = rows(out)
        outs.append((r, (tmp_path / name).read_bytes()))
    assert outs[0][0]["config_hash"] == outs[1][0]["config_hash"] and outs[0][1] == outs[1][1]
    replay = tmp_path / "replay.cfg"
    replay.write_text("".join(f"{k} = {outs[0][0][k]}\n" for k in RunConfig().as_dict()))
    code, out, _ = run(["solve", "--config", str(replay), "--out", str(tmp_path / "c.grid")], capsys)
    (r,) = rows(out)
    assert code == 0 and r["config_hash"] == outs[0][0]["config_hash"]
    assert (tmp_path / "c.grid").read_bytes() == outs[0][1]


def test_sweep_rows(capsys):
    code, out, _ = run(["sweep", "--grid", "12", "--block", "12,6,6", "--passes", "2",
                        "--sweep-t", "1,2", "--sweep-du", "0:2"], capsys)
    assert code == 0
    rs = rows(out)
    assert len(rs) == 6
    assert sum(r["status"].startswith("config_error") for r in rs) == 2
    assert sum(r["status"] == "ok" for r in rs) == 4


def test_bench_row(capsys):
    code, out, _ = run(["bench", "--kernel", "update", "--elements", "1000000", "--reps", "2"], capsys)
    (r,) = rows(out)
    assert code == 0 and r["kernel"] == "update" and float(r["bandwidth_Bps"]) > 0


def test_dist_inprocess_verify(tmp_path, capsys):
    code, out, _ = run(["dist", "--topo", "2,1,1", "--grid", "24", "--t", "2", "--block", "12,8,8",
                        "--cycles", "2", "--out-dir", str(tmp_path), "--verify"], capsys)
    assert code == 0
    rs = rows(out)
    assert len(rs) == 2 and all(r["verified"] == "bitwise match" for r in rs)
    assert (tmp_path / "rank_0.grid").exists() and (tmp_path / "rank_1.grid").exists()
    code, out, _ = run(["dist", "--topo", "1,1,4", "--grid", "32", "--t", "4", "--block", "32,8,8",
                        "--cycles", "3", "--verify"], capsys)
    assert code == 0 and all(r["verified"] == "bitwise match" for r in rows(out))
