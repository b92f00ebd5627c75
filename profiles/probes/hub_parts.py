"""Component times of the hybrid aggregation on a named shape at one K and T:
pack, hub GEMM (TFLOP/s over the 3-term product), tail SpMM."""
import sys, json, os
os.environ.setdefault("GNNC_HUB_FORMAT", "bf16x3")  # the probe packs bf16x3 terms
import torch
sys.path.insert(0, ".")
import paper_2306_15155_b200 as gc
from paper_2306_15155_b200 import graphs, hub, sparse, _native as nat
dev = torch.device("cuda", 0)
shape, K, T = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
g = gc.NormalizedGraph.from_adjacency(graphs.shape_graph(shape, device=dev))
a, d = g.a_tilde, g.d_inv_sqrt.to(dev)
x = torch.rand(a.n_rows, K, device=dev) - 0.5
plan = hub.hub_plan(a, T)
lib = nat.load(); st = torch.cuda.current_stream().cuda_stream
kp = lib.gc_hub_terms_rows(K)
bt = torch.empty(3 * kp * T, dtype=torch.bfloat16, device=dev)
sc = torch.empty(2, device=dev)
out = torch.empty(a.n_rows, K, device=dev)
def t_ms(fn, reps=10):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
    return sorted(ts)[reps // 2]
pack = lambda: nat.check(lib.gc_hub_pack(x.data_ptr(), K, K, plan.hub_cols.data_ptr(), T, d.data_ptr(), 0, bt.data_ptr(), sc.data_ptr(), st), "p")
gemm = lambda: nat.check(lib.gc_hub_gemm(plan.a_hub.data_ptr(), T, a.n_rows, T, bt.data_ptr(), K, 0, sc.data_ptr(), out.data_ptr(), K, d.data_ptr(), 0, st), "g")
tail = lambda: sparse._spmm(plan.tail, x, weighted=False, d_row=d, d_col=d, out=out, accumulate=True, timer=None)
r = {"shape": shape, "K": K, "T": T, "hub_edges_frac": plan.hub_edges / a.nnz}
r["pack_ms"] = t_ms(pack); r["gemm_ms"] = t_ms(gemm); r["tail_ms"] = t_ms(tail)
r["gemm_tflops"] = 2 * a.n_rows * T * K * 3 / r["gemm_ms"] / 1e9
r["a_hub_GBps"] = a.n_rows * T * 2 / r["gemm_ms"] / 1e6
xb = torch.randn(T, 3 * K, device=dev).to(torch.bfloat16)
r["cublas_bf16_proxy_ms"] = t_ms(lambda: plan.a_hub @ xb)
print(json.dumps(r))
