"""Drive the GAT layer (arxiv-shaped, K = 256, 1 head) for ncu captures of the
fused aggregation kernels: reuse/reassoc then reuse/sddmm, 3 calls each."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2306_15155_b200 as gc  # noqa: E402
from paper_2306_15155_b200 import graphs  # noqa: E402

dev = torch.device("cuda", 0)
at = gc.add_self_loops(graphs.shape_graph("arxiv", device=dev))
K = 256
h = torch.rand(at.n_rows, K, device=dev) - 0.5
w = torch.rand(K, K, device=dev) - 0.5
a_s, a_d = torch.rand(K, device=dev) - 0.5, torch.rand(K, device=dev) - 0.5
for form in ("reassoc", "sddmm"):
    spec = gc.GatLayerSpec(K, K, w, a_s, a_d, composition="reuse", attention=form)
    for _ in range(3):
        gc.gat_layer(at, h, spec)
torch.cuda.synchronize()
print("ok")
