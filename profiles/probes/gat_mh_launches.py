"""4-head GAT at K = 1024 on arxiv (TF32 class): reuse/reassoc and
recompute/reassoc layers for an ncu launch list (one warm call each, then
the profiled calls between cudaProfilerStart/Stop)."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import paper_2306_15155_b200 as gc  # noqa: E402
from paper_2306_15155_b200 import graphs  # noqa: E402

dev = torch.device("cuda", 0)
at = gc.add_self_loops(graphs.shape_graph("arxiv", device=dev))
K, H = 1024, 4
g = torch.Generator(device=dev)
g.manual_seed(7)
h = torch.rand(at.n_rows, K, device=dev, generator=g) - 0.5
w = torch.rand(K, K * H, device=dev, generator=g) - 0.5
a_s = torch.rand(K * H, device=dev, generator=g) - 0.5
a_d = torch.rand(K * H, device=dev, generator=g) - 0.5
specs = [gc.GatLayerSpec(K, K, w, a_s, a_d, composition=c, attention="reassoc", heads=H)
         for c in ("reuse", "recompute")]
for s in specs:
    gc.gat_layer(at, h, s)
torch.cuda.synchronize()
torch.cuda.profiler.start()
for s in specs:
    gc.gat_layer(at, h, s)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
