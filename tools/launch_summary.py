"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list: time per kernel name.

  python tools/launch_summary.py gpurun_out/launches_block.csv [--last N]
(--last N: only the last N launches, e.g. one steady-state frame)
"""
import csv
import re
import sys
from collections import defaultdict


def load(path):
    rows = []
    with open(path) as f:
        lines = [l for l in f if l.startswith('"')]
    for r in csv.DictReader(lines):
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        unit = r.get("Metric Unit", "ns")
        v = float(r["Metric Value"].replace(",", ""))
        scale = {"ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0, "nsecond": 1e-6}.get(unit, 1e-6)
        rows.append((int(r["ID"]), r["Kernel Name"], v * scale))
    rows.sort()
    return rows


def short(name):
    name = re.sub(r"\(.*", "", name)
    name = re.sub(r"^(void )?(mgpbd::)?(\(anonymous namespace\)::)?", "", name)
    return name


def main():
    path = sys.argv[1]
    last = int(sys.argv[sys.argv.index("--last") + 1]) if "--last" in sys.argv else 0
    rows = load(path)
    if last:
        rows = rows[-last:]
    agg = defaultdict(lambda: [0, 0.0])
    for _, name, ms in rows:
        k = short(name)
        agg[k][0] += 1
        agg[k][1] += ms
    tot = sum(v[1] for v in agg.values())
    print(f"{len(rows)} launches, {tot:.2f} ms total (serialised, cold-cache)")
    for k, (n, ms) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{ms:10.3f} ms {100 * ms / tot:6.2f}%  {n:7d}x  {1e3 * ms / n:9.2f} us  {k}")


if __name__ == "__main__":
    main()
