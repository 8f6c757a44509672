"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list: libcil kernels only,
grouped by kernel, with per-launch time and share of the libcil kernel time.
usage: python tools/launch_summary.py launches.csv "<command line>" > profiles/rNN_launches_summary.txt"""
import csv, re, sys
from collections import OrderedDict


def short(name):
    name = re.sub(r"\(.*$", "", name)             # drop the argument list
    name = name.replace("void ", "")
    return name


def main(path, cmd):
    agg = OrderedDict()
    lines = [l for l in open(path) if l.startswith('"')]      # drop the ==PROF== lines
    for r in csv.DictReader(lines):
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        k = r["Kernel Name"]
        if not any(t in k for t in ("cil::", "tc::", "g3::", "rd::")):
            continue
        k = short(k)
        us = float(r["Metric Value"]) / (1000.0 if r["Metric Unit"] == "ns" else 1.0)
        n, t = agg.get(k, (0, 0.0))
        agg[k] = (n + 1, t + us)
    tot = sum(t for _, t in agg.values())
    print(f"# ncu --metrics gpu__time_duration.sum --clock-control none, command: {cmd}")
    print("# cold-cache, serialised launches; libcil kernels only (warm-up + timed steps + e2e-free run)")
    print("# units: microseconds; share = fraction of libcil kernel time")
    for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{k[:44]:44s} launches={n:4d} total_us={t:10.1f} per_launch_us={t / n:10.1f} share={t / tot:6.3f}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "")
