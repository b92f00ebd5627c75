"""Reuse/reassoc GAT layer with and without the per-head fp16-row GEMM
epilogue path (gat._reuse_f16rows), interleaved, on the arxiv and products
shapes (TF32 class)."""
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import paper_2306_15155_b200 as gc  # noqa: E402
from paper_2306_15155_b200 import gat, graphs, profiling  # noqa: E402

dev = torch.device("cuda", 0)
real = gat._reuse_f16rows
for shape, cfgs in (("arxiv", ((1, 256), (4, 256), (4, 128))), ("products", ((1, 256),))):
    at = gc.add_self_loops(graphs.shape_graph(shape, device=dev))
    for heads, K in cfgs:
        g = torch.Generator(device=dev)
        g.manual_seed(K + heads)
        h = torch.rand(at.n_rows, K, device=dev, generator=g) - 0.5
        w = torch.rand(K, K * heads, device=dev, generator=g) - 0.5
        a_s = torch.rand(K * heads, device=dev, generator=g) - 0.5
        a_d = torch.rand(K * heads, device=dev, generator=g) - 0.5
        spec = gc.GatLayerSpec(K, K, w, a_s, a_d, composition="reuse", attention="reassoc",
                               heads=heads)
        row = {"shape": shape, "heads": heads, "K": K}
        for rnd in range(3):
            for name, fn in (("f16rows", real), ("pack", lambda *a: False)):
                gat._reuse_f16rows = fn
                med, _ = profiling.time_iterations(lambda: gc.gat_layer(at, h, spec), 3, 10)
                row.setdefault(name, []).append(round(med * 1e3, 4))
        gat._reuse_f16rows = real
        a = gc.gat_layer(at, h, spec)
        gat._reuse_f16rows = lambda *a: False
        b = gc.gat_layer(at, h, spec)
        gat._reuse_f16rows = real
        row["max_rel_diff"] = float(((a - b).norm() / b.norm()).item())
        print(json.dumps(row), flush=True)
