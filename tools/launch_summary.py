"""Summarise an ncu launch list (`ncu --metrics gpu__time_duration.sum[,dram__bytes_read.sum,
dram__bytes_write.sum] --csv --log-file X`): launches, mean time, share of GPU time and
DRAM bytes per launch for each kernel."""
import collections
import csv
import sys

TIME = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
BYTES = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}


def main(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr, rows = rows[0], rows[1:]
    ii, ki = hdr.index("ID"), hdr.index("Kernel Name")
    mi, vi, ui = hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    launches = collections.defaultdict(dict)
    for r in rows:
        v = float(r[vi].replace(",", ""))
        if r[mi] == "gpu__time_duration.sum":
            v *= TIME.get(r[ui], 1.0)
        else:
            v *= BYTES.get(r[ui], 1.0)
        launches[(int(r[ii]), r[ki])][r[mi]] = v
    agg = collections.defaultdict(lambda: {"n": 0, "us": 0.0, "bytes": 0.0})
    for (_, k), m in launches.items():
        a = agg[k.split("(")[0][:70]]
        a["n"] += 1
        a["us"] += m.get("gpu__time_duration.sum", 0.0)
        a["bytes"] += m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
    tot = sum(a["us"] for a in agg.values()) or 1.0
    print(f"{'kernel':70s} {'n':>5s} {'mean us':>10s} {'share':>7s} {'DRAM GB/launch':>15s}")
    for k, a in sorted(agg.items(), key=lambda x: -x[1]["us"]):
        print(f"{k:70s} {a['n']:5d} {a['us'] / a['n']:10.1f} {a['us'] / tot * 100:6.1f}% "
              f"{a['bytes'] / a['n'] / 1e9:15.4f}")


if __name__ == "__main__":
    main(sys.argv[1])
