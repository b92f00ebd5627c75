"""Summarise ncu --set full reports (.ncu-rep) into a markdown table: per
kernel launch the duration, DRAM bytes and rate, L2 hit rate and throughput,
achieved occupancy, and tensor-pipe activity, read with
`ncu -i <rep> --page raw --csv`.

    python profiles/summarize_ncu.py gpurun_out/ncu_r02/*.ncu-rep [--peak-gbs 6650]
"""

from __future__ import annotations

import argparse
import csv
import io
import subprocess
from pathlib import Path

NCU = "/usr/local/cuda/bin/ncu"
METRICS = {
    "dur_us": ("gpu__time_duration.sum", 1e-3),  # ns -> us
    "dram_rd": ("dram__bytes_read.sum", 1.0),
    "dram_wr": ("dram__bytes_write.sum", 1.0),
    "l2_hit": ("lts__t_sector_hit_rate.pct", 1.0),
    "l2_thru": ("lts__t_sectors.avg.pct_of_peak_sustained_elapsed", 1.0),
    "dram_thru": ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", 1.0),
    "occ": ("sm__warps_active.avg.pct_of_peak_sustained_active", 1.0),
    "sm_thru": ("sm__throughput.avg.pct_of_peak_sustained_elapsed", 1.0),
    "issue": ("sm__inst_issued.avg.pct_of_peak_sustained_active", 1.0),
    "regs": ("launch__registers_per_thread", 1.0),
    "utc": ("sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active", 1.0),
}
UNIT_SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1, "usecond": 1e3,
              "msecond": 1e6, "second": 1e9, "ns": 1, "us": 1e3, "ms": 1e6, "s": 1e9}


def rows_of(rep: Path) -> list[dict]:
    out = subprocess.run([NCU, "-i", str(rep), "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    data = list(csv.reader(io.StringIO(out)))
    hdr, units, body = data[0], data[1], data[2:]
    res = []
    for r in body:
        rec = {"kernel": r[hdr.index("Kernel Name")][:90], "id": r[hdr.index("ID")]}
        for key, (name, sc) in METRICS.items():
            if name not in hdr:
                continue
            i = hdr.index(name)
            try:
                v = float(r[i].replace(",", ""))
            except ValueError:
                continue
            rec[key] = v * UNIT_SCALE.get(units[i], 1.0) * sc
        res.append(rec)
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("reports", nargs="+")
    ap.add_argument("--peak-gbs", type=float, default=6650.0)
    args = ap.parse_args()
    print("| report | id | kernel | µs | DRAM rd+wr GB | DRAM GB/s (frac) | L2 hit % | L2 thru % "
          "| warps active % | regs | issue % | tensor % |")
    print("|---|---|---|---|---|---|---|---|---|---|---|---|")
    for rep in args.reports:
        for r in rows_of(Path(rep)):
            d = (r.get("dram_rd", 0) + r.get("dram_wr", 0))
            us = r.get("dur_us", 0)
            gbs = d / (us * 1e-6) / 1e9 if us else 0
            ten = r.get("utc", float("nan"))
            print(f"| {Path(rep).stem} | {r['id']} | `{r['kernel']}` | {us:.1f} | {d / 1e9:.3f} | "
                  f"{gbs:.0f} ({gbs / args.peak_gbs:.2f}) | {r.get('l2_hit', float('nan')):.1f} | "
                  f"{r.get('l2_thru', float('nan')):.1f} | {r.get('occ', float('nan')):.1f} | "
                  f"{r.get('regs', float('nan')):.0f} | {r.get('issue', float('nan')):.1f} | {ten:.1f} |")


if __name__ == "__main__":
    main()
