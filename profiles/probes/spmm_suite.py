"""Plain SpMM / hybrid times on the named shapes (A/B of builds via
GNNC_LIB_PATH)."""
import sys, json, os
import torch
sys.path.insert(0, ".")
import paper_2306_15155_b200 as gc
from paper_2306_15155_b200 import graphs, hub, sparse
dev = torch.device("cuda", 0)
def t_ms(fn, reps=7):
    for _ in range(2): fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
    return sorted(ts)[reps // 2]
res = {"lib": os.environ.get("GNNC_LIB_PATH", "default")}
for shape in ("arxiv", "reddit", "products"):
    g = gc.NormalizedGraph.from_adjacency(graphs.shape_graph(shape, device=dev)).with_precomputed()
    a, d = g.a_tilde, g.d_inv_sqrt.to(dev)
    for K in (32, 256):
        x = torch.rand(a.n_rows, K, device=dev) - 0.5
        out = torch.empty(a.n_rows, K, device=dev)
        res[f"{shape}/K{K}/plain_weighted"] = round(t_ms(lambda: sparse.spmm(g.n_tilde, x, out=out)), 4)
        res[f"{shape}/K{K}/plain_dyn"] = round(t_ms(lambda: sparse.spmm_unweighted(a, x, d_col=d, d_row=d, out=out)), 4)
        if shape == "reddit" and K == 256:
            spec = ("stair", 15)
            res[f"{shape}/K{K}/stair15"] = round(t_ms(lambda: hub.hybrid_aggregate(a, x, d, spec, out=out)), 4)
            res[f"{shape}/K{K}/stair15_tail"] = round(t_ms(lambda: hub.tail_part(a, x, d, spec, out, d_row=d)), 4)
    del g, a
print(json.dumps(res))
