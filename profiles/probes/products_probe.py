"""One products-shaped GCN aggregation at K for ncu (precompute Ñ SpMM)."""
import sys
import torch
sys.path.insert(0, ".")
import paper_2306_15155_b200 as gc
from paper_2306_15155_b200 import graphs, sparse
dev = torch.device("cuda", 0)
K = int(sys.argv[1]) if len(sys.argv) > 1 else 256
g = gc.NormalizedGraph.from_adjacency(graphs.shape_graph("products", device=dev)).with_precomputed()
x = torch.rand(g.a_tilde.n_rows, K, device=dev)
for _ in range(3):
    sparse.spmm(g.n_tilde, x)
torch.cuda.synchronize()
