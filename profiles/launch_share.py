#!/usr/bin/env python
"""Per-kernel launch statistics from an ncu launch list
(--metrics gpu__time_duration.sum --csv), e.g. gpurun_out/launches_<tag>.csv."""
import csv
import sys
from collections import defaultdict


def main(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, mi, vi, ui = (h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"),
                      h.index("Metric Unit"))
    t = defaultdict(list)
    unit = None
    for r in rows[hi + 1:]:
        if len(r) > vi and r[mi] == "gpu__time_duration.sum":
            t[r[ki]].append(float(r[vi].replace(",", "")))
            unit = r[ui]
    scale = {"ns": 1e-6, "us": 1e-3, "ms": 1.0}.get(unit, 1.0)
    total = sum(sum(v) for v in t.values())
    print(f"{'launches':>8} {'mean ms':>10} {'total ms':>10} {'share':>7}  kernel")
    for k, v in sorted(t.items(), key=lambda kv: -sum(kv[1])):
        print(f"{len(v):8d} {sum(v) / len(v) * scale:10.3f} {sum(v) * scale:10.2f} "
              f"{sum(v) / total:7.1%}  {k[:90]}")


if __name__ == "__main__":
    main(sys.argv[1])
