"""Attribute ncu per-instruction execution counts to CUDA source lines.

    python tools/sass_lines.py <report.ncu-rep> <libsp200.so> [--top N] [--kernel REGEX]

ncu's source page needs the sources on the profiling box; this joins its SASS
page (address -> instructions executed, stall samples) with the line table of
the same binary (nvdisasm -g on the cubin extracted from the .so), so it must
be run against the exact .so that was profiled.
"""
import argparse
import collections
import csv
import io
import os
import re
import subprocess
import tempfile


def sass_csv(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True, check=True).stdout
    lines = out.splitlines()
    kernel = next(csv.reader([lines[0]]))[1]
    rows = list(csv.DictReader(io.StringIO("\n".join(lines[1:]))))
    return kernel, rows


def line_table(so, mangled_hint):
    tmp = tempfile.mkdtemp()
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(so)], cwd=tmp, capture_output=True)
    table = {}
    for f in sorted(os.listdir(tmp)):
        if not f.endswith(".cubin"):
            continue
        txt = subprocess.run(["nvdisasm", "-g", os.path.join(tmp, f)], capture_output=True, text=True).stdout
        cur_fn, cur_line = None, None
        for ln in txt.splitlines():
            m = re.match(r"\.text\.(\S+):$", ln.strip())
            if m:
                cur_fn = m.group(1)
                table.setdefault(cur_fn, {})
                continue
            m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
            if m:
                cur_line = f"{os.path.basename(m.group(1))}:{m.group(2)}"
                continue
            m = re.match(r"\s*/\*([0-9a-f]+)\*/\s+\S", ln)
            if m and cur_fn:
                table[cur_fn][int(m.group(1), 16)] = cur_line
    return table


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("so")
    ap.add_argument("--top", type=int, default=40)
    ap.add_argument("--mangled", default=None, help="mangled kernel name (default: match by template args)")
    a = ap.parse_args()
    kernel, rows = sass_csv(a.rep)
    table = line_table(a.so, kernel)
    # map the demangled "k_temporal<(int)4, (int)32, ..., (bool)1>" to a mangled entry
    args = re.findall(r"\((?:int|bool)\)(\d+)", kernel)
    cands = [k for k in table if "k_temporal" in k or "k_sweep1" in k]
    if a.mangled:
        fn = a.mangled
    else:
        def sig(m):
            return re.findall(r"L[ib](\d+)E", m)
        fn = next(k for k in cands if sig(k) == args and ("k_temporal" in kernel) == ("k_temporal" in k))
    lt = table[fn]
    base = min(int(r["Address"], 16) for r in rows)
    per_line = collections.Counter()
    stall = collections.Counter()
    ops = collections.defaultdict(collections.Counter)
    total = 0
    for r in rows:
        off = int(r["Address"], 16) - base
        ln = lt.get(off, "?")
        n = int(r["Instructions Executed"] or 0)
        per_line[ln] += n
        total += n
        stall[ln] += int(r["Warp Stall Sampling (All Samples)"] or 0)
        op = r["Source"].split()[0] if r["Source"].split() else "?"
        if op.startswith("@"):
            op = r["Source"].split()[1]
        ops[ln][op.split(".")[0]] += n
    stot = sum(stall.values()) or 1
    print(f"{fn}\ntotal warp instructions {total:,}")
    for ln, n in per_line.most_common(a.top):
        top_ops = ", ".join(f"{o}:{c * 100 // max(n, 1)}%" for o, c in ops[ln].most_common(4))
        print(f"{ln:28s} {n / total * 100:6.2f}% inst  {stall[ln] / stot * 100:6.2f}% stall  {top_ops}")


if __name__ == "__main__":
    main()
