"""One launch of every GAT-path kernel (and the products SpMM) inside a
cudaProfilerStart/Stop range, for `ncu --profile-from-start off`:
arxiv-shaped RMAT, K in {32, 256, 1024}, 1 and 4 heads — the fused
aggregations (gat_aggregate, gat_sddmm_aggregate), the API-path attention
(node_proj + edge_softmax; attn_score + edge_softmax), and the products-shape
GCN aggregation at K = 256.  Warm-up (autotuners, plans) happens outside the
range.  Prints the algorithmic bytes per launch per kernel.

    python profiles/probes/gat_ncu.py [--ks 32,256,1024] [--products]
"""
import argparse
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import paper_2306_15155_b200 as gc  # noqa: E402
from paper_2306_15155_b200 import graphs  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--ks", default="32,256,1024")
ap.add_argument("--heads", default="1,4")
ap.add_argument("--products", action="store_true")
args = ap.parse_args()
dev = torch.device("cuda", 0)
at = gc.add_self_loops(graphs.shape_graph("arxiv", device=dev))
n, m = at.n_rows, at.nnz
model = {}
work = []
for heads in (int(h) for h in args.heads.split(",")):
    for K in (int(k) for k in args.ks.split(",")):
        if heads > 1 and K > 256:
            continue
        g = torch.Generator(device=dev)
        g.manual_seed(K)
        h = torch.rand(n, K, device=dev, generator=g) - 0.5
        w = torch.rand(K, K * heads, device=dev, generator=g) - 0.5
        a_s = torch.rand(K * heads, device=dev, generator=g) - 0.5
        a_d = torch.rand(K * heads, device=dev, generator=g) - 0.5
        for comp in ("reuse:reassoc", "reuse:sddmm"):
            spec = gc.GatLayerSpec(K, K, w, a_s, a_d, composition=comp.split(":")[0],
                                   attention=comp.split(":")[1], heads=heads)
            work.append((f"gat_layer {comp} heads={heads} K={K}",
                         (lambda s=spec, hh=h: gc.gat_layer(at, hh, s))))
            hw = gc.gemm(h, w)
            work.append((f"atten_calc {comp.split(':')[1]} heads={heads} K={K}",
                         (lambda s=spec, x=hw: gc.atten_calc(at, x, s))))
        # algorithmic bytes per launch (edge-gather model, fp32, int32)
        model[f"heads={heads} K={K}"] = {
            "gat_aggregate": 4 * (n + 1) + 4 * m + 4 * m + 4 * m * K + 4 * n * K + 4 * n,
            "gat_sddmm_aggregate": 4 * (n + 1) + 4 * m + 4 * m * K + 4 * n * K + 4 * n * K,
            "edge_softmax": 4 * (n + 1) + 4 * m + 4 * n + 4 * m + 4 * m,
            "attn_score": 4 * (n + 1) + 4 * m + 4 * m * K + 4 * n * K + 4 * m}
for name, fn in work:  # warm: plans, variant autotuners
    fn()
    fn()
torch.cuda.synchronize()
if args.products:
    a = graphs.shape_graph("products", device=dev)
    gp = gc.NormalizedGraph.from_adjacency(a)
    del a
    hp = torch.rand(gp.a_tilde.n_rows, 256, device=dev) - 0.5
    wp = torch.rand(256, 256, device=dev) - 0.5
    spec = gc.GcnLayerSpec(256, 256, wp, composition="dynamic", order="update_first")
    for _ in range(3):
        gc.gcn_layer(gp, hp, spec)
    work.append(("products gcn dynamic:update_first K=256", lambda: gc.gcn_layer(gp, hp, spec)))
torch.cuda.synchronize()
torch.cuda.profiler.start()
for name, fn in work:
    torch.cuda.nvtx.range_push(name)
    fn()
    torch.cuda.nvtx.range_pop()
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print(json.dumps({"order": [w[0] for w in work], "alg_bytes": model, "n": n, "m": m}))
