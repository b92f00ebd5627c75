"""GAT on the arxiv shape: ms per layer for every (composition, attention)
pair at heads 1/4 and K 32/256/1024 (CUDA events, median of 10)."""
import sys, json
import numpy as np, torch
sys.path.insert(0, ".")
import paper_2306_15155_b200 as gc
from paper_2306_15155_b200 import graphs, profiling, sparse
dev = torch.device("cuda", 0)
a = sparse.add_self_loops(graphs.shape_graph(sys.argv[1] if len(sys.argv) > 1 else "arxiv", device=dev))
def t_ms(fn, reps=10):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
    return sorted(ts)[reps // 2]
for heads, K in ((1, 32), (1, 256), (1, 1024), (4, 32), (4, 256)):
    rng = np.random.default_rng(0)
    h = torch.from_numpy(rng.uniform(-.5, .5, (a.n_rows, K)).astype(np.float32)).to(dev)
    w = rng.uniform(-.5, .5, (K, heads * K)).astype(np.float32)
    asr = rng.uniform(-.5, .5, heads * K).astype(np.float32); ads = rng.uniform(-.5, .5, heads * K).astype(np.float32)
    row = {"heads": heads, "K": K}
    for comp in ("reuse", "recompute"):
        for att in ("reassoc", "sddmm"):
            spec = gc.GatLayerSpec(K, K, w, asr, ads, composition=comp, heads=heads, attention=att)
            row[f"{comp}:{att}"] = round(t_ms(lambda: gc.gat_layer(a, h, spec)), 4)
    # the alpha-materialising SDDMM attention alone
    hw = torch.rand(a.n_rows, heads * K, device=dev)
    spec = gc.GatLayerSpec(K, K, w, asr, ads, heads=heads, attention="sddmm")
    row["atten_calc_sddmm"] = round(t_ms(lambda: gc.atten_calc(a, hw, spec)), 4)
    spec = gc.GatLayerSpec(K, K, w, asr, ads, heads=heads, attention="reassoc")
    row["atten_calc_reassoc"] = round(t_ms(lambda: gc.atten_calc(a, hw, spec)), 4)
    print(json.dumps(row), flush=True)
