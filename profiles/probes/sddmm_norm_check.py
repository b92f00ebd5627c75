import sys, torch, time
sys.path.insert(0, ".")
import paper_2306_15155_b200 as gc
from paper_2306_15155_b200 import graphs, sparse
dev = torch.device("cuda", 0)
for shape in ("arxiv", "products"):
    a = sparse.add_self_loops(graphs.shape_graph(shape, device=dev))
    d = sparse.inv_sqrt_degrees(a).to(dev)
    t0 = time.time(); v = sparse.sddmm_norm(a, d); torch.cuda.synchronize()
    ref = d[a.row_of_nnz()] * d[a.col_idx.long()]
    print(shape, "ok", bool(torch.equal(v.values if hasattr(v, "values") else v, ref)), time.time() - t0, flush=True)
