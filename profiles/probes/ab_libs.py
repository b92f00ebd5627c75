"""A/B of libgnnc builds (GNNC_LIB_PATH) on the bench step: for each library
and shape, one short bench.py run (no sweep / extras / CPU), reporting the
step time and the per-kernel CUDA-event times.

    python profiles/probes/ab_libs.py --libs a.so,b.so --shapes reddit,products [--k 256]
    python profiles/probes/ab_libs.py --libs default,env:GNNC_HUB_SPLIT=stair:8:10
"""
import argparse
import json
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]
ap = argparse.ArgumentParser()
ap.add_argument("--libs", required=True)
ap.add_argument("--shapes", default="reddit")
ap.add_argument("--k", default="256")
ap.add_argument("--rounds", type=int, default=2)
ap.add_argument("--extra", default="")
args = ap.parse_args()
res = []
for rnd in range(args.rounds):
    for shape in args.shapes.split(","):
        for k in args.k.split(","):
            for lib in args.libs.split(","):
                env = dict(os.environ)
                if lib.startswith("env:"):  # env:KEY=VAL+KEY=VAL on the default library
                    env.update(kv.split("=", 1) for kv in lib[4:].split("+"))
                elif lib != "default":
                    env["GNNC_LIB_PATH"] = str(Path(lib).resolve())
                out = f"/tmp/ab_{os.getpid()}.json"
                cmd = [sys.executable, str(ROOT / "bench.py"), "--shape", shape, "--k", k, "--steps", "20",
                       "--warmup", "3", "--no-sweep", "--no-extra", "--no-cpu", "--no-fp32-class",
                       "--out", out] + (args.extra.split() if args.extra else [])
                r = subprocess.run(cmd, env=env, capture_output=True, text=True, cwd=ROOT)
                if r.returncode:
                    print(lib, shape, k, "FAILED", r.stderr[-800:], flush=True)
                    continue
                d = json.loads(Path(out).read_text())
                row = {"round": rnd, "lib": lib, "shape": shape, "K": int(k), "ms": d["ms_per_step"],
                       "kernel_ms": d["kernel_ms"], "split": d["dense_split"]["chosen"],
                       "variant": d["spmm_variant"]["chosen"], "parity": d["parity"]["rel_err"],
                       "sm_mhz": d["clocks"]["sm_mhz"]}
                print(json.dumps(row), flush=True)
                res.append(row)
Path(ROOT / "gpurun_out").mkdir(exist_ok=True)
(ROOT / "gpurun_out" / "ab_libs.json").write_text(json.dumps(res, indent=1))
