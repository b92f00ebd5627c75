"""GAT layer ms per composition on the arxiv and products shapes (TF32
class), for A/B of GNNC_HALF_GATHER (set in the environment)."""
import json
import os
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import paper_2306_15155_b200 as gc  # noqa: E402
from paper_2306_15155_b200 import graphs, profiling, selector  # noqa: E402

dev = torch.device("cuda", 0)
out = []
for shape, ks in (("arxiv", (32, 256, 1024)), ("products", (32, 256))):
    at = gc.add_self_loops(graphs.shape_graph(shape, device=dev))
    for K in ks:
        g = torch.Generator(device=dev)
        g.manual_seed(K)
        h = torch.rand(at.n_rows, K, device=dev, generator=g) - 0.5
        w = torch.rand(K, K, device=dev, generator=g) - 0.5
        a_s = torch.rand(K, device=dev, generator=g) - 0.5
        a_d = torch.rand(K, device=dev, generator=g) - 0.5
        row = {"shape": shape, "K": K, "half": os.environ.get("GNNC_HALF_GATHER", "1")}
        for c in selector.B200_COMPOSITIONS["gat"]:
            spec = gc.GatLayerSpec(K, K, w, a_s, a_d, composition=c.split(":")[0],
                                   attention=c.split(":")[1])
            med, _ = profiling.time_iterations(lambda: gc.gat_layer(at, h, spec), 3, 10)
            row[c] = round(med * 1e3, 4)
        print(json.dumps(row), flush=True)
        out.append(row)
    del at
    torch.cuda.empty_cache()
