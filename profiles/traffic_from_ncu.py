#!/usr/bin/env python
"""Writes profiles/ncu_traffic.json from an ncu --set full report of one
bp_kernel launch: dram__bytes_read.sum + dram__bytes_write.sum per launch
(bench.py reports it as roofline.traffic)."""
import csv
import io
import json
import os
import subprocess
import sys

rep, workload, mode = sys.argv[1], sys.argv[2], sys.argv[3]
extra = dict(a.split("=", 1) for a in sys.argv[4:])  # e.g. projections_per_launch=64
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True,
                     check=True).stdout
rows = list(csv.reader(io.StringIO(out)))
d = {h: (u, v) for h, u, v in zip(rows[0], rows[1], rows[2])}
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
tot = 0.0
for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
    u, v = d[k]
    tot += float(v) * scale[u]
path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "ncu_traffic.json")
data = json.load(open(path)) if os.path.exists(path) else {}
kname = d.get("Kernel Name", ("", ""))[1]
short = kname.split("(")[0].split("<")[0].split()[-1].split("::")[-1]
entry = {"dram_bytes_per_launch": tot, "kernel": kname, "source": os.path.basename(rep)}
entry.update({k: int(v) if v.isdigit() else v for k, v in extra.items()})
data[f"{workload}/{mode}/{short}"] = entry
json.dump(data, open(path, "w"), indent=1)
print(data)
