"""Per-kernel times of the edge-wise kernels (Ñ SDDMM, edge softmax, SDDMM
attention) on the named shapes, with their algorithmic bytes -> GB/s."""
import sys, json
import numpy as np, torch
sys.path.insert(0, ".")
import paper_2306_15155_b200 as gc
from paper_2306_15155_b200 import graphs, sparse, _native as nat
dev = torch.device("cuda", 0)

def t_ms(fn, reps=10):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
    return sorted(ts)[reps // 2]

for shape in sys.argv[1:] or ["arxiv", "reddit", "products"]:
    a = sparse.add_self_loops(graphs.shape_graph(shape, device=dev))
    n, m = a.n_rows, a.nnz
    d = sparse.inv_sqrt_degrees(a).to(dev)
    res = {"shape": shape, "n": n, "m": m, "max_deg": int((a.row_ptr[1:] - a.row_ptr[:-1]).max()),
           "heavy_rows": int(a.softmax_heavy_rows().numel())}
    ms = t_ms(lambda: sparse.sddmm_norm(a, d))
    byt = 4 * (n + 1) + 4 * m * 4  # row_ptr, col, values, d_j gather, out
    res["sddmm_norm"] = {"ms": round(ms, 4), "GB/s": round(byt / ms / 1e6, 1)}
    lib = nat.load()
    st = torch.cuda.current_stream().cuda_stream
    for H in (1, 4):
        s = torch.rand(H, n, device=dev); t = torch.rand(H, n, device=dev)
        alpha = torch.empty(H, m, device=dev)
        hv = a.softmax_heavy_rows()
        def sm(heavy=True):
            nat.check(lib.gc_edge_softmax_f32(a.row_ptr.data_ptr(), a.col_idx.data_ptr(), s.data_ptr(),
                                              t.data_ptr(), H, 0.2, n, m, hv.data_ptr() if heavy else None,
                                              hv.numel() if heavy else 0, alpha.data_ptr(), st), "sm")
        ms = t_ms(sm); ms0 = t_ms(lambda: sm(False))
        byt = 4 * (n + 1) + 4 * m + 4 * H * n + 4 * H * m * 2
        res[f"edge_softmax_h{H}"] = {"ms": round(ms, 4), "GB/s": round(byt / ms / 1e6, 1),
                                     "ms_without_heavy_ctas": round(ms0, 4)}
        for K in (32, 256):
            hw = torch.rand(n, H * K, device=dev)
            spec = gc.GatLayerSpec(K, K, np.zeros((K, H * K)), np.ones(H * K), np.ones(H * K), heads=H,
                                   attention="sddmm")
            ms = t_ms(lambda: gc.atten_calc(a, hw, spec))
            byt = 4 * (n + 1) + 4 * m + 4 * m * H * K + 4 * n * H * K + 4 * H * m
            res[f"attn_sddmm_h{H}_k{K}"] = {"ms": round(ms, 4), "GB/s_edge_gather": round(byt / ms / 1e6, 1)}
            del hw
    print(json.dumps(res), flush=True)
    del a
