"""Collect ncu per-launch DRAM traffic of the SpMM (profiles/run_ncu_traffic.sh
output) into profiles/traffic.json, keyed like bench.py's roofline lookup."""

import csv
import json
import sys
from pathlib import Path

src = Path(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/ncu_traffic")
out = {}
for f in sorted(src.glob("*.csv")):
    rows = list(csv.reader(f.open()))
    hi = next(i for i, r in enumerate(rows) if "Metric Name" in r)
    hdr, data = rows[hi], rows[hi + 1:]
    mi, vi, ui = hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    vals = {}
    for r in data:
        v = float(r[vi].replace(",", ""))
        vals[r[mi]] = v * scale.get(r[ui], 1)
    comp = f.stem.replace("_", ":", 1)
    comp = comp.replace("precompute:", "precompute:").replace("dynamic:", "dynamic:")
    out[f"reddit/K256/{comp}"] = int(vals["dram__bytes_read.sum"] + vals["dram__bytes_write.sum"])
    out[f"reddit/K256/{comp}/detail"] = vals
Path("profiles/traffic.json").write_text(json.dumps(out, indent=1) + "\n")
print(json.dumps(out, indent=1))
