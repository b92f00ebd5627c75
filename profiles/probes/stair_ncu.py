"""One staircase dense-part launch on Reddit (for ncu)."""
import sys
import torch
sys.path.insert(0, ".")
import paper_2306_15155_b200 as gc
from paper_2306_15155_b200 import graphs, hub
dev = torch.device("cuda", 0)
K = int(sys.argv[1]) if len(sys.argv) > 1 else 256
spec = hub._parse_spec(sys.argv[2] if len(sys.argv) > 2 else "stair:18:10")
g = gc.NormalizedGraph.from_adjacency(graphs.shape_graph("reddit", device=dev))
a, d = g.a_tilde, g.d_inv_sqrt.to(dev)
x = torch.rand(a.n_rows, K, device=dev) - 0.5
out = torch.empty(a.n_rows, K, device=dev)
packed = hub.pack(a, x, d, spec)
for _ in range(3):
    hub.dense_part(a, x, d, spec, out, d_row=d, packed=packed)
torch.cuda.synchronize()
