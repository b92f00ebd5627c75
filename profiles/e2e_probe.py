"""Where does the end-to-end (host in / host out) GCN layer time go?

Times, on the Reddit-shaped graph at K = 256: the bare H2D / D2H of the layer
operands, the device-resident layer, and the host-pipelined public-API layer
for several row-block counts.  Wall clock around a synchronised loop (this is
what bench.py's ``e2e`` measures).  Prints one JSON document.
"""

from __future__ import annotations

import json
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import paper_2306_15155_b200 as gc  # noqa: E402
from paper_2306_15155_b200 import gcn, graphs  # noqa: E402


def wall(fn, reps=5, warm=2):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        ts.append((time.perf_counter() - t0) * 1e3)
    return float(np.median(ts))


def main():
    dev = torch.device("cuda", 0)
    K = 256
    A = graphs.shape_graph("reddit", device=dev)
    g = gc.NormalizedGraph.from_adjacency(A).with_precomputed()
    del A
    n = g.a_tilde.n_rows
    h_pin = (torch.rand(n, K) - 0.5).pin_memory()
    h_dev = h_pin.to(dev)
    out_pin = torch.empty(n, K, pin_memory=True)
    res = {"n": n, "K": K, "bytes": n * K * 4}
    res["h2d_ms"] = wall(lambda: h_dev.copy_(h_pin, non_blocking=True))
    res["d2h_ms"] = wall(lambda: out_pin.copy_(h_dev, non_blocking=True))
    for comp in ("dynamic:aggregate_first", "precompute:aggregate_first"):
        base, order = comp.split(":")
        spec = gc.GcnLayerSpec(K, K, torch.rand(K, K, device=dev) - 0.5, composition=base, order=order)
        r = {"device_layer_ms": wall(lambda: gc.gcn_layer(g, h_dev, spec))}
        r["unpipelined_ms"] = wall(lambda: gc.gcn_layer(g, h_dev.cpu().pin_memory() if False else h_pin.to(dev), spec).cpu())
        for blocks in (1, 2, 4, 8, 16):
            gcn.HOST_PIPELINE_BLOCKS = blocks
            r[f"pipelined_{blocks}_ms"] = wall(lambda: gc.gcn_layer(g, h_pin, spec))
        res[comp] = r
        print(json.dumps({comp: r}), file=sys.stderr, flush=True)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
