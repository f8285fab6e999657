"""Aggregate an ncu --csv launch list (gpu__time_duration.sum) by kernel name."""

import csv
import re
import sys
from collections import defaultdict


def short(name: str) -> str:
    name = re.sub(r"\(.*", "", name)
    name = re.sub(r"void |spectre::", "", name)
    return name[:60]


def main(path):
    rows = []
    with open(path) as f:
        lines = [ln for ln in f if not ln.startswith("==")]
    rd = csv.DictReader(lines)
    for r in rd:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "ns")
        ns = v * {"ns": 1, "usecond": 1e3, "us": 1e3, "msecond": 1e6, "ms": 1e6}.get(unit, 1)
        rows.append((short(r["Kernel Name"]), r.get("Grid Size", ""), ns))
    agg = defaultdict(lambda: [0, 0.0])
    for k, g, ns in rows:
        agg[k][0] += 1
        agg[k][1] += ns
    total = sum(v[1] for v in agg.values())
    print(f"{len(rows)} launches, total {total / 1e6:.3f} ms")
    for k, (n, ns) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{ns / 1e6:9.3f} ms {100 * ns / total:5.1f}%  n={n:5d}  avg={ns / n / 1e3:8.2f} us  {k}")


if __name__ == "__main__":
    main(sys.argv[1])
