"""GCN layer times per composition on a named shape at K (device path)."""
import sys, json
import numpy as np, torch
sys.path.insert(0, ".")
import paper_2306_15155_b200 as gc
from paper_2306_15155_b200 import graphs
dev = torch.device("cuda", 0)
shape, K = sys.argv[1], int(sys.argv[2])
g = gc.NormalizedGraph.from_adjacency(graphs.shape_graph(shape, device=dev)).with_precomputed()
h = torch.rand(g.a_tilde.n_rows, K, device=dev) - 0.5
w = np.random.default_rng(0).uniform(-.5, .5, (K, K)).astype(np.float32)
res = {"shape": shape, "K": K}
for comp in ("precompute:aggregate_first", "precompute:update_first", "dynamic:aggregate_first", "dynamic:update_first"):
    base, order = comp.split(":")
    spec = gc.GcnLayerSpec(K, K, w, composition=base, order=order)
    for _ in range(3): gc.gcn_layer(g, h, spec)
    torch.cuda.synchronize()
    ts = []
    for _ in range(7):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); gc.gcn_layer(g, h, spec); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
    res[comp] = round(sorted(ts)[3], 4)
print(json.dumps(res))
