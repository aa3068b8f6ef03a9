"""CPU: the analytical models (sp/perfmodel.py) on the shipped B200 files,
against the reference's own functions evaluated on the same files
(tests/golden/perfmodel.json, made by tests/golden/make_golden_perfmodel.py),
plus the format errors of pkg/tests/test_perfmodel.py."""

import json
import os

import pytest

from paper_1006_3148_b200 import perfmodel as pm

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "perfmodel.json")))


@pytest.fixture(scope="module")
def b200():
    return pm.load_machine_model("b200")


@pytest.fixture(scope="module")
def nvl():
    return pm.load_network_model("nvlink5")


def test_baselines_match_reference(b200):
    assert "b200" in pm.shipped_machine_names()
    assert pm.baseline_perf(b200) == GOLD["baseline_perf"]
    assert abs(pm.baseline_perf(b200) / 1e9 - 409.3) < 1e-9  # the HBM roofline line of bench.py
    for t, v in GOLD["pipelined_bound"].items():
        assert pm.pipelined_bound(b200, int(t)) == v
    with pytest.raises(ValueError):
        pm.pipelined_bound(b200, 0)


def test_cycle_model_matches_reference(b200):
    for level, exp in GOLD["cache_cycle_model"].items():
        r = pm.cache_cycle_model(b200, "jacobi", level)
        assert [r.cycles_min, r.cycles_max, r.bytes_per_update, r.bandwidth_min, r.bandwidth_max] == exp
    assert pm.default_bj(b200) == GOLD["bj_L2"]
    for t, (req, ok) in GOLD["l3_scalability_check"].items():
        assert list(pm.l3_scalability_check(b200, int(t), GOLD["bj_L2"])) == [req, ok]
    with pytest.raises(ValueError):
        pm.cache_cycle_model(b200, "nope", "L2")
    with pytest.raises(ValueError):
        pm.cache_cycle_model(b200, "jacobi", "L7")


def test_halo_model_matches_reference(nvl):
    for key, v in GOLD["multihalo_advantage"].items():
        L, h = (int(x) for x in key.split(","))
        assert pm.multihalo_advantage(L, h, nvl) == v
        assert pm.comm_efficiency(L, h, nvl) == GOLD["comm_efficiency"][key]
    with pytest.raises(ValueError):
        pm.comm_efficiency(0, 1, nvl)


def test_format_errors(tmp_path):
    with pytest.raises(pm.ModelFormatError):
        pm.parse_machine_model("name = x\nbogus line\n")
    with pytest.raises(pm.ModelFormatError):
        pm.parse_machine_model("name = x\nfreq_hz = 1\n")  # missing fields
    with pytest.raises(pm.ModelFormatError):
        pm.parse_network_model("latency_s = -1\nbandwidth_Bps = 1\nnode_perf_lups = 1\n")
    text = open(os.path.join(pm.DATA_DIR, "b200.model")).read()
    with pytest.raises(pm.ModelFormatError):
        pm.parse_machine_model(text.replace("m_uc1 = 88.9e9", "m_uc1 = 1.0e9"))
    with pytest.raises(pm.ModelFormatError):
        pm.parse_machine_model(text + "\njacobi.L2.colour = red\n")
    p = tmp_path / "m.model"
    p.write_text(text)
    assert pm.load_machine_model(str(p)).name == "NVIDIA B200"
