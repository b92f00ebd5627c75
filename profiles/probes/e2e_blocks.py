"""e2e (pinned host H in, pinned host output out) of the Reddit K=256 layer
for several row-block counts of the host pipeline."""
import sys, json, time
import numpy as np, torch
sys.path.insert(0, ".")
import paper_2306_15155_b200 as gc
from paper_2306_15155_b200 import gcn, graphs, profiling
dev = torch.device("cuda", 0)
K = int(sys.argv[1]) if len(sys.argv) > 1 else 256
g = gc.NormalizedGraph.from_adjacency(graphs.shape_graph("reddit", device=dev)).with_precomputed()
rng = profiling.config_rng(0, "reddit", K, K)
inp = profiling.draw_inputs(rng, g.a_tilde.n_rows, K, K, "gcn")
h = torch.from_numpy(inp["h"].astype(np.float32)).pin_memory()
for comp in sys.argv[2].split(",") if len(sys.argv) > 2 else ["precompute:update_first"]:
    base, order = comp.split(":")
    spec = gc.GcnLayerSpec(K, K, inp["w"].astype(np.float32), composition=base, order=order)
    row = {"K": K, "comp": comp}
    for k in (-1, 0, 4, 6):
        gcn.HOST_PIPELINE_BLOCKS = k
        for _ in range(3): gc.gcn_layer(g, h, spec)
        torch.cuda.synchronize()
        ts = []
        for _ in range(8):
            t0 = time.perf_counter(); gc.gcn_layer(g, h, spec); ts.append(time.perf_counter() - t0)
        row[f"blocks={k}"] = round(float(np.median(ts)) * 1e3, 3)
    print(json.dumps(row), flush=True)
