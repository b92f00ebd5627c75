"""Autotuner candidate timings (ms) per graph shape and K for the SpMM and the
fused GAT aggregations: which lane-group shape / hub tags win where."""
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2306_15155_b200 as gc  # noqa: E402
from paper_2306_15155_b200 import graphs, sparse  # noqa: E402
from paper_2306_15155_b200.gat import _projections  # noqa: E402

dev = torch.device("cuda", 0)
out = {}
for shape in ("arxiv", "products", "reddit"):
    at = gc.add_self_loops(graphs.shape_graph(shape, device=dev))
    d = gc.inv_sqrt_degrees(at).to(dev)
    for K in (32, 64, 128, 256):
        h = torch.rand(at.n_rows, K, device=dev) - 0.5
        gc.spmm_unweighted(at, h, d_row=d, d_col=d)
        spec = gc.GatLayerSpec(K, K, torch.eye(K, device=dev), torch.rand(K, device=dev) - 0.5,
                               torch.rand(K, device=dev) - 0.5)
        s, t = _projections(h, spec, spec.attn_src, spec.attn_dst, K, K)
        sparse.gat_aggregate(at, s[0], t[0], 0.2, h)
        sparse.gat_sddmm_aggregate(at, spec.attn_src, spec.attn_dst, 0.2, h)
        out[f"{shape}/K{K}"] = {m: at._plans.get(("variant", m, K, "times")) for m in ("spmm", "gat", "gatsd")}
        out[f"{shape}/K{K}"]["chosen"] = {m: at._plans.get(("variant", m, K)) for m in ("spmm", "gat", "gatsd")}
        print(json.dumps({f"{shape}/K{K}": out[f"{shape}/K{K}"]}), file=sys.stderr, flush=True)
        del h
    del at
    torch.cuda.empty_cache()
print(json.dumps(out))
