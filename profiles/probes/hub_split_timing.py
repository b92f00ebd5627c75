"""Hybrid aggregation (hub block on tcgen05 + sparse tail) vs plain SpMM on a
named shape: the autotuner's timings per T, per composition and K, plus a
row-sampled parity check against the plain SpMM."""
import sys, json
import torch
sys.path.insert(0, ".")
import paper_2306_15155_b200 as gc
from paper_2306_15155_b200 import graphs, hub, sparse
dev = torch.device("cuda", 0)
shape = sys.argv[1] if len(sys.argv) > 1 else "reddit"
Ks = [int(k) for k in (sys.argv[2].split(",") if len(sys.argv) > 2 else ["32", "256", "1024"])]
g = gc.NormalizedGraph.from_adjacency(graphs.shape_graph(shape, device=dev)).with_precomputed()
a, d = g.a_tilde, g.d_inv_sqrt.to(dev)
for K in Ks:
    x = torch.rand(a.n_rows, K, device=dev) - 0.5
    for pre in (False, True):
        vals = g.n_tilde.values if pre else None
        T = hub.choose_split(a, x, d, values=vals)
        times = a._plans[("hubsplit-choice", K, pre, "times")] if ("hubsplit-choice", K, pre, "times") in a._plans else None
        row = {"shape": shape, "K": K, "composition": "precompute" if pre else "dynamic", "chosen_T": T, "ms": times}
        if T:
            ref = sparse.spmm(g.n_tilde, x) if pre else sparse.spmm_unweighted(a, x, d_col=d, d_row=d)
            out = hub.hybrid_aggregate(a, x, d, T, values=vals)
            row["rel_err_vs_plain"] = float((out - ref).abs().max() / ref.abs().max())
        print(json.dumps(row), flush=True)
    del x
