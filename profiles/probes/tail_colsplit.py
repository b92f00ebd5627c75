"""Does splitting the tail SpMM into column-range passes (each pass gathers
from an L2-sized slice of X) beat one pass?"""
import sys, json
import torch
sys.path.insert(0, ".")
import paper_2306_15155_b200 as gc
from paper_2306_15155_b200 import graphs, hub, sparse
from paper_2306_15155_b200.sparse import CsrMatrix
dev = torch.device("cuda", 0)
K = int(sys.argv[1]) if len(sys.argv) > 1 else 256
g = gc.NormalizedGraph.from_adjacency(graphs.shape_graph("reddit", device=dev))
a, d = g.a_tilde, g.d_inv_sqrt.to(dev)
x = torch.rand(a.n_rows, K, device=dev) - 0.5
spec = hub._parse_spec(sys.argv[2]) if len(sys.argv) > 2 else ("stair", 18, 10)
plan = hub.hub_plan(a, spec)
tail = plan.tail
out = torch.zeros(a.n_rows, K, device=dev)
def t_ms(fn, reps=7):
    for _ in range(2): fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
    return sorted(ts)[reps // 2]
rows = tail.row_of_nnz()
col = tail.col_idx.long()
def split(parts):
    bounds = [a.n_cols * i // parts for i in range(parts + 1)]
    res = []
    for p in range(parts):
        m = (col >= bounds[p]) & (col < bounds[p + 1])
        cnt = torch.bincount(rows[m], minlength=a.n_rows)
        rp = torch.zeros(a.n_rows + 1, dtype=torch.int32, device=dev); rp[1:] = torch.cumsum(cnt, 0).int()
        c = CsrMatrix(a.n_rows, a.n_cols, rp, tail.col_idx[m].contiguous(), torch.ones(int(m.sum()), device=dev), validate=False)
        c._unit = True
        res.append(c)
    return res
r = {"K": K, "tail_edges": tail.nnz}
r["1pass"] = t_ms(lambda: sparse._spmm(tail, x, weighted=False, d_row=d, d_col=d, out=out, accumulate=True, timer=None))
for parts in (2, 3, 4):
    ps = split(parts)
    def run(ps=ps):
        for p in ps:
            sparse._spmm(p, x, weighted=False, d_row=d, d_col=d, out=out, accumulate=True, timer=None)
    r[f"{parts}pass"] = t_ms(run)
print(json.dumps(r))
