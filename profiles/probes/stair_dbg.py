"""Dense-part time under GNNC_HUB_DBG modes (bottleneck hunt; results wrong)."""
import sys, json, os
import torch
sys.path.insert(0, ".")
import paper_2306_15155_b200 as gc
from paper_2306_15155_b200 import graphs, hub
dev = torch.device("cuda", 0)
g = gc.NormalizedGraph.from_adjacency(graphs.shape_graph("reddit", device=dev))
a, d = g.a_tilde, g.d_inv_sqrt.to(dev)
x = torch.rand(a.n_rows, 256, device=dev) - 0.5
out = torch.empty(a.n_rows, 256, device=dev)
spec = ("stair", 18, 10)
packed = hub.pack(a, x, d, spec)
def t_ms(fn, reps=7):
    for _ in range(2): fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
    return sorted(ts)[reps // 2]
print(json.dumps({"dbg": os.environ.get("GNNC_HUB_DBG", "0"), "dense_ms": t_ms(lambda: hub.dense_part(a, x, d, spec, out, d_row=d, packed=packed))}))
