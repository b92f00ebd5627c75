"""One edge softmax (1 head) and one Ñ SDDMM on a named shape, for ncu."""
import sys
import torch
sys.path.insert(0, ".")
from paper_2306_15155_b200 import graphs, sparse, _native as nat
dev = torch.device("cuda", 0)
a = sparse.add_self_loops(graphs.shape_graph(sys.argv[1] if len(sys.argv) > 1 else "products", device=dev))
n, m = a.n_rows, a.nnz
d = sparse.inv_sqrt_degrees(a).to(dev)
s = torch.rand(1, n, device=dev); t = torch.rand(1, n, device=dev)
alpha = torch.empty(1, m, device=dev)
hv = a.softmax_heavy_rows()
lib = nat.load(); st = torch.cuda.current_stream().cuda_stream
for _ in range(2):
    nat.check(lib.gc_edge_softmax_f32(a.row_ptr.data_ptr(), a.col_idx.data_ptr(), s.data_ptr(), t.data_ptr(), 1, 0.2, n, m,
                                      hv.data_ptr(), hv.numel(), alpha.data_ptr(), st), "sm")
    sparse.sddmm_norm(a, d)
torch.cuda.synchronize()
