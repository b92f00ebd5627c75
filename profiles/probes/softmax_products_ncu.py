"""One edge-softmax launch on the products shape (heavy-row list on), for an
ncu --set full capture of edge_softmax_kernel."""
import sys
import torch
sys.path.insert(0, ".")
from paper_2306_15155_b200 import graphs, sparse, _native as nat
dev = torch.device("cuda", 0)
a = sparse.add_self_loops(graphs.shape_graph(sys.argv[1] if len(sys.argv) > 1 else "products", device=dev))
n, m = a.n_rows, a.nnz
lib = nat.load()
s = torch.rand(1, n, device=dev)
t = torch.rand(1, n, device=dev)
alpha = torch.empty(1, m, device=dev)
hv = a.softmax_heavy_rows()
for _ in range(3):
    nat.check(lib.gc_edge_softmax_f32(a.row_ptr.data_ptr(), a.col_idx.data_ptr(), s.data_ptr(),
                                      t.data_ptr(), 1, 0.2, n, m, hv.data_ptr(), hv.numel(),
                                      alpha.data_ptr(), torch.cuda.current_stream().cuda_stream), "sm")
torch.cuda.synchronize()
print("done", n, m, hv.numel())
