"""Summarise an ncu launch list (--metrics gpu__time_duration.sum,dram__bytes_*
--csv): per kernel name, launches, mean time, share of the total, mean DRAM
bytes.  Usage: python profiles/scripts/launch_summary.py launches.csv [steps]"""
import csv
import sys
from collections import defaultdict

SCALE = {"ns": 1.0, "us": 1e3, "usecond": 1e3, "ms": 1e6, "msecond": 1e6, "nsecond": 1.0,
         "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}
rows = [r for r in csv.reader(open(sys.argv[1])) if r and not r[0].startswith("==")]
if rows and "Kernel Name" in rows[0]:
    h = rows.pop(0)
    idi, ki, mi, ui, vi = (h.index(x) for x in ("ID", "Kernel Name", "Metric Name", "Metric Unit",
                                               "Metric Value"))
else:  # headerless --log-file output: ID, PID, process, host, kernel, ..., metric, unit, value
    idi, ki, mi, ui, vi = 0, 4, 12, 13, 14
per = defaultdict(dict)
for r in rows:
    if len(r) <= vi:
        continue
    per[(r[idi], r[ki])][r[mi]] = float(r[vi].replace(",", "")) * SCALE.get(r[ui], 1.0)
agg = defaultdict(lambda: [0, 0.0, 0.0])
for (_, name), m in per.items():
    short = name.split("(")[0].replace("void ", "").replace("(anonymous namespace)::", "")
    a = agg[short]
    a[0] += 1
    a[1] += m.get("gpu__time_duration.sum", 0.0)
    a[2] += m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
tot = sum(a[1] for a in agg.values())
print("| kernel | launches | time / launch | share | DRAM / launch |")
print("|---|---|---|---|---|")
for k, (n, t, b) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"| `{k[:90]}` | {n} | {t / n / 1e3:.1f} us | {100 * t / tot:.1f} % | {b / n / 1e9:.3f} GB |")
