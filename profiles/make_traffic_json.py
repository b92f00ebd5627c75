"""Launch-list summary and profiles/traffic.json from an ncu launch list
(`profiles/run_ncu_r02.sh`: --metrics gpu__time_duration.sum,
dram__bytes_read.sum, dram__bytes_write.sum over the bench's timed steps).

Prints a markdown table (per kernel: launches, µs per launch, share of the
profiled steps, DRAM GB per launch) and records, for the bench's roofline
lookup, the DRAM bytes per launch of the dominant SpMM (the tail of the dense
split when one is chosen) under the key bench.py uses:
  "<shape>/K<K>/<composition>[/tail/<split>]".

    python profiles/make_traffic_json.py gpurun_out/ncu_r02 [--shape reddit --k 256]
"""

from __future__ import annotations

import argparse
import csv
import json
from collections import OrderedDict
from pathlib import Path


def launches(path: Path) -> list[dict]:
    rows = list(csv.reader(path.open()))
    hi = next(i for i, r in enumerate(rows) if "Metric Name" in r)
    hdr = rows[hi]
    col = {k: hdr.index(k) for k in ("ID", "Kernel Name", "Metric Name", "Metric Value")}
    by_id: "OrderedDict[str, dict]" = OrderedDict()
    for r in rows[hi + 1:]:
        if len(r) < len(hdr):
            continue
        rec = by_id.setdefault(r[col["ID"]], {"kernel": r[col["Kernel Name"]]})
        rec[r[col["Metric Name"]]] = float(r[col["Metric Value"]].replace(",", ""))
    return list(by_id.values())


def short(name: str) -> str:
    name = name.replace("unnamed>::", "").replace("void ", "")
    return name.split("(")[0]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("src")
    ap.add_argument("--shape", default="reddit")
    ap.add_argument("--k", type=int, default=256)
    ap.add_argument("--steps", type=int, default=2)
    args = ap.parse_args()
    src = Path(args.src)
    recs = launches(src / "launches.csv")
    forced = (src / "forced.txt").read_text().split() if (src / "forced.txt").exists() else []
    split = next((f.split("=")[1] for f in forced if f.startswith("split=")), "0")
    comp = next((f.split("=")[1] for f in forced if f.startswith("composition=")), "")
    total = sum(r.get("gpu__time_duration.sum", 0) for r in recs)
    agg: "OrderedDict[str, list]" = OrderedDict()
    for r in recs:
        agg.setdefault(short(r["kernel"]), []).append(r)
    print(f"forced: split={split} composition={comp}; {len(recs)} launches over {args.steps} steps\n")
    print("| kernel | launches | µs / launch | share | DRAM GB / launch |")
    print("|---|---|---|---|---|")
    for k, rs in sorted(agg.items(), key=lambda kv: -sum(x.get("gpu__time_duration.sum", 0)
                                                          for x in kv[1])):
        t = sum(x.get("gpu__time_duration.sum", 0) for x in rs)
        d = sum(x.get("dram__bytes_read.sum", 0) + x.get("dram__bytes_write.sum", 0) for x in rs)
        print(f"| `{k}` | {len(rs)} | {t / len(rs) / 1e3:.1f} | {t / total:.3f} | "
              f"{d / len(rs) / 1e9:.3f} |")
    spmm = [r for r in recs if short(r["kernel"]).startswith("spmm_kernel")]
    if not spmm:
        return
    dram = [int(r.get("dram__bytes_read.sum", 0) + r.get("dram__bytes_write.sum", 0)) for r in spmm]
    key = f"{args.shape}/K{args.k}/{comp}" + (f"/tail/{split}" if split not in ("0", "") else "")
    out_p = Path("profiles/traffic.json")
    data = json.loads(out_p.read_text()) if out_p.exists() else {}
    data[key] = int(sum(dram) / len(dram))
    data[key + "/source"] = str(src / "launches.csv")
    # L2 side of the same kernel from the --set full capture (if present):
    # bytes through the L2 slices and ncu's L2 / L1 throughput fractions
    full = src / "spmm_tail_reddit_k256.raw.csv.gz"
    if full.exists():
        import gzip
        rows = list(csv.reader(gzip.open(full, "rt")))
        hdr, r = rows[0], rows[2]
        get = lambda k: float(r[hdr.index(k)].replace(",", ""))  # noqa: E731
        data[key + "/l2"] = {
            "l2_bytes": int(get("lts__t_sectors.sum") * 32),
            "lts_throughput_pct": round(get("lts__throughput.avg.pct_of_peak_sustained_elapsed"), 1),
            "l1tex_throughput_pct": round(get("l1tex__throughput.avg.pct_of_peak_sustained_active"), 1),
            "l2_hit_pct": round(get("lts__t_sector_hit_rate.pct"), 1),
            "warps_active_pct": round(get("sm__warps_active.avg.pct_of_peak_sustained_active"), 1),
            "kernel_us": round(get("gpu__time_duration.sum"), 1),
            "source": str(full)}
    out_p.write_text(json.dumps(data, indent=1) + "\n")
    print(f"\n{key}: {data[key]} DRAM bytes per launch (mean of {len(dram)})")


if __name__ == "__main__":
    main()
