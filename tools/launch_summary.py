"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv).

python tools/launch_summary.py gpurun_out/launches.csv "command line" > profiles/rNN_launches_summary.txt
"""
import csv
import re
import sys
from collections import OrderedDict


def short(name):
    name = re.sub(r"\(.*$", "", name) if not name.startswith("cub::") else name
    name = re.sub(r"^void ", "", name)
    name = re.sub(r"amrx::(\(anonymous namespace\)|<unnamed>)::", "", name)
    return name


def main():
    path = sys.argv[1]
    cmd = sys.argv[2] if len(sys.argv) > 2 else ""
    rows = []
    with open(path) as f:
        lines = [ln for ln in f if ln.startswith('"')]
    for r in csv.DictReader(lines):
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "ns")
        ms = v * {"ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0,
                  "nsecond": 1e-6, "second": 1e3}.get(unit, 1e-6)
        rows.append((short(r["Kernel Name"]), ms))
    agg = OrderedDict()
    for k, ms in rows:
        t, n = agg.get(k, (0.0, 0))
        agg[k] = (t + ms, n + 1)
    total = sum(t for t, _ in agg.values())
    print("ncu --metrics gpu__time_duration.sum --clock-control none (cold-cache, serialised launches)")
    if cmd:
        print("command:", cmd)
    print()
    for k, (t, n) in sorted(agg.items(), key=lambda kv: -kv[1][0]):
        print(f"{t:10.3f} ms  {100 * t / total:5.1f}%  x {n:2d}  {k}")
    print(f"\ntotal {total:.3f} ms over {len(rows)} launches")


if __name__ == "__main__":
    main()
