"""Update-first GCN layers at K = 512 / 1024 (Reddit, products) and 4-head
reuse GAT at K = 1024 (arxiv) with the GEMM epilogue emitting chunked-scale
fp16 rows (sparse.F16ROWS_CHUNKED) vs fp32 product + per-row pack,
interleaved CUDA-event medians."""
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import paper_2306_15155_b200 as gc  # noqa: E402
from paper_2306_15155_b200 import graphs, profiling, sparse  # noqa: E402

dev = torch.device("cuda", 0)


def bench(fn):
    row = {}
    for _ in range(3):
        for name, on in (("chunked", True), ("pack", False)):
            sparse.F16ROWS_CHUNKED = on
            med, _ = profiling.time_iterations(fn, 3, 7)
            row.setdefault(name, []).append(round(med * 1e3, 4))
    sparse.F16ROWS_CHUNKED = True
    return row


for shape, ks in (("reddit", (512, 1024)), ("products", (512, 1024))):
    g = gc.NormalizedGraph.from_adjacency(graphs.shape_graph(shape, device=dev)).with_precomputed()
    for K in ks:
        gen = torch.Generator(device=dev)
        gen.manual_seed(K)
        h = torch.rand(g.a_tilde.n_rows, K, device=dev, generator=gen) - 0.5
        w = torch.rand(K, K, device=dev, generator=gen) - 0.5
        spec = gc.GcnLayerSpec(K, K, w, composition="dynamic", order="update_first")
        r = {"shape": shape, "K": K, "layer": "gcn dynamic:update_first"}
        r.update(bench(lambda: gc.gcn_layer(g, h, spec)))
        print(json.dumps(r), flush=True)
        del h, w
    del g
    torch.cuda.empty_cache()
at = gc.add_self_loops(graphs.shape_graph("arxiv", device=dev))
K, H = 1024, 4
gen = torch.Generator(device=dev)
gen.manual_seed(7)
h = torch.rand(at.n_rows, K, device=dev, generator=gen) - 0.5
w = torch.rand(K, K * H, device=dev, generator=gen) - 0.5
a_s = torch.rand(K * H, device=dev, generator=gen) - 0.5
a_d = torch.rand(K * H, device=dev, generator=gen) - 0.5
for comp in ("reuse", "recompute"):
    spec = gc.GatLayerSpec(K, K, w, a_s, a_d, composition=comp, attention="reassoc", heads=H)
    r = {"shape": "arxiv", "K": K, "heads": H, "layer": f"gat {comp}:reassoc"}
    r.update(bench(lambda: gc.gat_layer(at, h, spec)))
    print(json.dumps(r), flush=True)
