"""Host enqueue time vs device time of one GCN layer (Reddit K=256): is the
step host-bound?  Also per-primitive host costs."""
import sys, time, json
import numpy as np, torch
sys.path.insert(0, ".")
import paper_2306_15155_b200 as gc
from paper_2306_15155_b200 import graphs, hub, sparse
dev = torch.device("cuda", 0)
K = 256
g = gc.NormalizedGraph.from_adjacency(graphs.shape_graph("reddit", device=dev)).with_precomputed()
h = torch.rand(g.a_tilde.n_rows, K, device=dev) - 0.5
spec = gc.GcnLayerSpec(K, K, np.random.default_rng(0).uniform(-.5, .5, (K, K)).astype(np.float32),
                       composition="dynamic", order="update_first")
for _ in range(3): gc.gcn_layer(g, h, spec)
torch.cuda.synchronize()
N = 20
t0 = time.perf_counter()
for _ in range(N): gc.gcn_layer(g, h, spec)
t1 = time.perf_counter()
torch.cuda.synchronize()
t2 = time.perf_counter()
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(N): gc.gcn_layer(g, h, spec)
e1.record(); torch.cuda.synchronize()
res = {"host_enqueue_ms_per_layer": (t1 - t0) / N * 1e3, "wall_ms_per_layer": (t2 - t0) / N * 1e3,
       "device_ms_per_layer": e0.elapsed_time(e1) / N}
# per-piece host cost
a, d = g.a_tilde, g.d_inv_sqrt.to(dev)
hw = sparse.gemm(h, spec.weights)
split = hub.choose_split(a, hw, d)
def host(fn, n=50):
    torch.cuda.synchronize(); t = time.perf_counter()
    for _ in range(n): fn()
    t = (time.perf_counter() - t) / n * 1e3
    torch.cuda.synchronize(); return t
out = torch.empty_like(hw)
packed = hub.pack(a, hw, d, split)
res["host_gemm_ms"] = host(lambda: sparse.gemm(h, spec.weights))
res["host_pack_ms"] = host(lambda: hub.pack(a, hw, d, split))
res["host_dense_ms"] = host(lambda: hub.dense_part(a, hw, d, split, out, d_row=d, packed=packed))
res["host_tail_ms"] = host(lambda: hub.tail_part(a, hw, d, split, out, d_row=d, relu=True))
res["split"] = hub.spec_label(split)
print(json.dumps(res))
