"""Multi-head GAT (reuse, reassociated attention) on the arxiv shape: all heads
in one fused pass over the pattern (gat_aggregate_mh) vs one fused pass per
head, ms per layer (CUDA events, median of 20 after 3 warmups)."""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2306_15155_b200 as gc
from paper_2306_15155_b200 import gat as gat_mod
from paper_2306_15155_b200 import graphs

dev = torch.device("cuda", 0)
shape = sys.argv[1] if len(sys.argv) > 1 else "arxiv"
a = gc.add_self_loops(graphs.shape_graph(shape, device=dev))


def t_ms(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return sorted(ts)[reps // 2]


rng = np.random.default_rng(0)
for heads, k in ((4, 32), (4, 64), (4, 256), (8, 32)):
    h = torch.from_numpy(rng.uniform(-0.5, 0.5, (a.n_rows, k)).astype(np.float32)).to(dev)
    w = rng.uniform(-0.5, 0.5, (k, heads * k)).astype(np.float32)
    a_s = rng.uniform(-0.5, 0.5, heads * k).astype(np.float32)
    a_d = rng.uniform(-0.5, 0.5, heads * k).astype(np.float32)
    spec = gc.GatLayerSpec(k, k, w, a_s, a_d, heads=heads, composition="reuse")
    r = {"shape": shape, "heads": heads, "k1": k, "k2": k}
    outs = {}
    for mode in (False, True):
        gat_mod.MULTIHEAD_ONE_PASS = mode
        r["one_pass_ms" if mode else "per_head_ms"] = round(t_ms(lambda: gc.gat_layer(a, h, spec)), 4)
        outs[mode] = gc.gat_layer(a, h, spec)
    r["max_abs_diff"] = float((outs[True] - outs[False]).abs().max())
    print(json.dumps(r), flush=True)
