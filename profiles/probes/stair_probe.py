"""Staircase plans on a named shape: steps, covered edges, cells, and the
dense-part / tail times per δ, vs the best block plan and the plain SpMM."""
import sys, json
import torch
sys.path.insert(0, ".")
import paper_2306_15155_b200 as gc
from paper_2306_15155_b200 import graphs, hub, sparse, _native as nat
dev = torch.device("cuda", 0)
shape = sys.argv[1] if len(sys.argv) > 1 else "reddit"
K = int(sys.argv[2]) if len(sys.argv) > 2 else 256
g = gc.NormalizedGraph.from_adjacency(graphs.shape_graph(shape, device=dev))
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
ref = sparse.spmm_unweighted(a, x, d_col=d, d_row=d)
print(json.dumps({"plain_ms": t_ms(lambda: sparse.spmm_unweighted(a, x, d_col=d, d_row=d, out=out))}), flush=True)
specs = [hub._parse_spec(x) for x in sys.argv[3].split(",")] if len(sys.argv) > 3 else \
    [4096, ("stair", 12, 10), ("stair", 18, 10), ("stair", 18, 15), ("stair", 18, 20), ("stair", 12, 20)]
for spec in specs:
    try:
        plan = hub.hub_plan(a, spec)
    except ValueError as e:
        print(spec, e); continue
    bt = hub.pack(a, x, d, spec)
    r = {"spec": hub.spec_label(spec), "steps": getattr(plan, "steps", None), "dense_edges": plan.hub_edges,
         "tail_edges": plan.tail.nnz, "cells": plan.cells}
    r["pack_ms"] = t_ms(lambda: hub.pack(a, x, d, spec))
    r["dense_ms"] = t_ms(lambda: hub.dense_part(a, x, d, spec, out, d_row=d, packed=bt))
    r["tail_ms"] = t_ms(lambda: hub.tail_part(a, x, d, spec, out, d_row=d))
    r["total_ms"] = t_ms(lambda: hub.hybrid_aggregate(a, x, d, spec, out=out))
    y = hub.hybrid_aggregate(a, x, d, spec)
    r["rel_err_vs_plain"] = float((y - ref).abs().max() / ref.abs().max())
    r["dense_tflops"] = 2 * plan.cells * K * hub.term_count() / r["dense_ms"] / 1e9; r["terms"] = hub.term_count()
    print(json.dumps(r), flush=True)
    a._plans.pop(("hubsplit", hub._parse_spec(spec)), None)
