"""One SDDMM-form attention (atten_calc) on a named shape, for ncu."""
import sys
import numpy as np, torch
sys.path.insert(0, ".")
import paper_2306_15155_b200 as gc
from paper_2306_15155_b200 import graphs, sparse
dev = torch.device("cuda", 0)
shape, K, H = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
a = sparse.add_self_loops(graphs.shape_graph(shape, device=dev))
hw = torch.rand(a.n_rows, H * K, device=dev)
spec = gc.GatLayerSpec(K, K, np.zeros((K, H * K)), np.ones(H * K), np.ones(H * K), heads=H, attention="sddmm")
for _ in range(2):
    gc.atten_calc(a, hw, spec)
torch.cuda.synchronize()
