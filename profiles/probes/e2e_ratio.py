"""e2e (pinned host H in, pinned host output out) of the Reddit K=256 layer
for several values of the host pipeline's cost-model constant
E2E_ROW_EDGE_RATIO (D2H seconds per output row over aggregation seconds per
edge), which places the two-block split."""
import json
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2306_15155_b200 as gc  # noqa: E402
from paper_2306_15155_b200 import gcn, graphs, profiling  # noqa: E402

dev = torch.device("cuda", 0)
K = 256
g = gc.NormalizedGraph.from_adjacency(graphs.shape_graph("reddit", device=dev)).with_precomputed()
rng = profiling.config_rng(0, "reddit", K, K)
inp = profiling.draw_inputs(rng, g.a_tilde.n_rows, K, K, "gcn")
h = torch.from_numpy(inp["h"].astype(np.float32)).pin_memory()
spec = gc.GcnLayerSpec(K, K, inp["w"].astype(np.float32), composition="dynamic", order="update_first")
res = []
for rnd in range(2):
    for ratio in (400.0, 800.0, 1200.0, 1700.0, 2500.0, 4000.0):
        gcn.E2E_ROW_EDGE_RATIO = ratio
        g.__dict__.pop("_row_block_cache", None)
        for _ in range(3):
            gc.gcn_layer(g, h, spec)
        torch.cuda.synchronize()
        ts = []
        for _ in range(10):
            t0 = time.perf_counter()
            gc.gcn_layer(g, h, spec)
            ts.append(time.perf_counter() - t0)
        blocks = [(lo, hi) for lo, hi, _ in g._row_block_cache[next(iter(g._row_block_cache))]]
        row = {"round": rnd, "ratio": ratio, "ms": round(float(np.median(ts)) * 1e3, 3), "blocks": blocks}
        print(json.dumps(row), flush=True)
        res.append(row)
json.dump(res, open("gpurun_out/e2e_ratio.json", "w"), indent=1)
