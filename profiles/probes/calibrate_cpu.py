"""Calibrate the CPU baseline: the oracle's C/OpenMP port of the reference
kernels vs the reference itself (gnncompose, numba + OpenBLAS), same graph,
same inputs, same thread count, in THIS (build) container — the reference
cannot travel to the GPU box (/root/reference is absent there).

Writes profiles/data/cpu_calibration.json: per config the median layer time
of each (3 reps after 1 warm-up; the reference's first call includes numba
JIT, excluded by the warm-up) and ratio = port_time / reference_time.
bench.py reports the ratio next to its CPU numbers.

    python profiles/probes/calibrate_cpu.py [--shapes arxiv,reddit] [--ks 32,256]
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, "/root/reference/pkg/src")
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")


def median_time(fn, reps=3):
    fn()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    return float(np.median(ts))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shapes", default="arxiv,reddit")
    ap.add_argument("--ks", default="32,256")
    args = ap.parse_args()

    import gnncompose as ref
    from gnncompose import runtime
    from oracle import gnn_oracle as orc
    from paper_2306_15155_b200 import graphs, profiling

    threads = runtime.configure_threads(os.cpu_count())
    orc.set_threads(threads)
    out = {"threads": threads, "cpu": next((ln.split(":", 1)[1].strip() for ln in
                                            Path("/proc/cpuinfo").read_text().splitlines()
                                            if ln.startswith("model name")), "unknown"),
           "reference": "gnncompose 0.1.0 (numba %s) from /root/reference" % __import__("numba").__version__,
           "composition": "dynamic, heuristic order (aggregate_first at k1 == k2)", "rows": []}
    for shape in args.shapes.split(","):
        a = graphs.shape_graph(shape, device="cpu")
        rp, ci, v = a.numpy()
        del a
        ra = ref.CsrMatrix(n_rows=rp.size - 1, n_cols=rp.size - 1, row_ptr=rp, col_idx=ci, values=v)
        rg = ref.NormalizedGraph.from_adjacency(ra)
        og = orc.GcnGraph.from_adjacency(orc.Csr(rp.size - 1, rp.size - 1, rp, ci, v))
        assert np.array_equal(rg.a_tilde.col_idx, og.a_tilde.col_idx)
        n = rp.size - 1
        for K in (int(k) for k in args.ks.split(",")):
            inp = profiling.draw_inputs(profiling.config_rng(0, shape, K, K), n, K, K, "gcn")
            h = inp["h"].astype(np.float32).astype(np.float64)
            w = inp["w"].astype(np.float32).astype(np.float64)
            spec = ref.GcnLayerSpec(K, K, w)
            t_ref = median_time(lambda: ref.gcn_layer(rg, h, spec))
            t_port = median_time(lambda: orc.gcn_layer(og, h, w, "dynamic"))
            r_out = ref.gcn_layer(rg, h, spec)
            p_out = orc.gcn_layer(og, h, w, "dynamic")
            row = {"shape": shape, "K": K, "m_tilde": int(og.a_tilde.nnz),
                   "reference_s": round(t_ref, 4), "port_s": round(t_port, 4),
                   "port_over_reference": round(t_port / t_ref, 3),
                   "reference_edges_per_s": round(og.a_tilde.nnz / t_ref, 1),
                   "port_edges_per_s": round(og.a_tilde.nnz / t_port, 1),
                   "max_abs_diff": float(np.abs(r_out - p_out).max())}
            print(json.dumps(row), flush=True)
            out["rows"].append(row)
    dst = ROOT / "profiles" / "data" / "cpu_calibration.json"
    dst.write_text(json.dumps(out, indent=1) + "\n")
    print(dst)


if __name__ == "__main__":
    main()
