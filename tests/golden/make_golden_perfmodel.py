"""Generate tests/golden/perfmodel.json: the REFERENCE's analytical models
(sp/perfmodel.py) evaluated on this repo's B200 model files.

    python tests/golden/make_golden_perfmodel.py    (build container only: needs /root/reference)

The reference's parser reads our flat-format files, so the fixture pins both
the file format and the model arithmetic of paper_1006_3148_b200/perfmodel.py.
"""
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
DATA = os.path.join(HERE, "..", "..", "paper_1006_3148_b200", "data")


def main():
    sys.path.insert(0, "/root/reference/pkg/src")
    from stencilpipe import perfmodel as pm  # read-only import of the reference

    m = pm.parse_machine_model(open(os.path.join(DATA, "b200.model")).read())
    net = pm.parse_network_model(open(os.path.join(DATA, "nvlink5.network")).read())
    out = {"machine": "b200", "network": "nvlink5",
           "baseline_perf": pm.baseline_perf(m),
           "pipelined_bound": {t: pm.pipelined_bound(m, t) for t in range(1, 9)},
           "cache_cycle_model": {}, "l3_scalability_check": {}, "multihalo_advantage": {},
           "comm_efficiency": {}}
    for level in ("smem", "L2", "HBM"):
        r = pm.cache_cycle_model(m, "jacobi", level)
        out["cache_cycle_model"][level] = [r.cycles_min, r.cycles_max, r.bytes_per_update,
                                           r.bandwidth_min, r.bandwidth_max]
    bj = pm.cache_cycle_model(m, "jacobi", "L2").bandwidth_min
    out["bj_L2"] = bj
    for t in range(0, 9):
        req, ok = pm.l3_scalability_check(m, t, bj)
        out["l3_scalability_check"][t] = [req, ok]
    for L in (16, 64, 256, 512, 1024):
        for h in (1, 2, 4, 8, 16):
            key = f"{L},{h}"
            out["multihalo_advantage"][key] = pm.multihalo_advantage(L, h, net)
            out["comm_efficiency"][key] = pm.comm_efficiency(L, h, net)
    from stencilpipe.cli import RunConfig  # config hash of the CLI rows (sp/cli.py:71-74)
    out["cli_config_hash"] = {
        "default": RunConfig().config_hash(), "d_u=7": RunConfig(d_u=7).config_hash(),
        "grid16_t2_compressed": RunConfig(nx=16, ny=16, nz=16, t=2, bx=16, by=8, bz=8,
                                          mode="compressed").config_hash()}
    with open(os.path.join(HERE, "perfmodel.json"), "w") as f:
        json.dump(out, f, indent=1)
    print("wrote perfmodel.json")


if __name__ == "__main__":
    main()
