"""Staircase band ratio / δ sweep on Reddit (aggregation time, f16x2)."""
import sys, json
import torch
sys.path.insert(0, ".")
import paper_2306_15155_b200 as gc
from paper_2306_15155_b200 import graphs, hub
dev = torch.device("cuda", 0)
K = int(sys.argv[1]) if len(sys.argv) > 1 else 256
g = gc.NormalizedGraph.from_adjacency(graphs.shape_graph("reddit", device=dev))
a, d = g.a_tilde, g.d_inv_sqrt.to(dev)
x = torch.rand(a.n_rows, K, device=dev) - 0.5
out = torch.empty(a.n_rows, K, device=dev)
def t_ms(fn, reps=7):
    for _ in range(2): fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
    return sorted(ts)[reps // 2]
for ratio in (2 ** 0.5, 2 ** 0.25):
    hub.STAIR_BAND_RATIO = ratio
    for dl in (0.005, 0.008, 0.012):
        spec = ("stair", int(dl * 1000), 10)
        a._plans.pop(("hubsplit", spec), None)
        plan = hub.hub_plan(a, spec)
        ms = t_ms(lambda: hub.hybrid_aggregate(a, x, d, spec, out=out))
        print(json.dumps({"ratio": round(ratio, 3), "delta": dl, "steps": len(plan.steps), "cells": plan.cells,
                          "dense_edges": plan.hub_edges, "ms": round(ms, 4)}), flush=True)
        a._plans.pop(("hubsplit", spec), None)
