"""Does the hub GEMM overlap the tail SpMM on a side stream?  Times
sequential (GEMM then tail with ACCUMULATE) against concurrent (GEMM on a
side stream into its own buffer, tail on the main stream, then a combine)."""
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
lib = nat.load()
kp = lib.gc_hub_terms_rows(K)
bt = torch.empty(3 * kp * T, dtype=torch.bfloat16, device=dev)
sc = torch.empty(2, device=dev)
out = torch.empty(a.n_rows, K, device=dev); ch = torch.empty_like(out)
side = torch.cuda.Stream(dev)
def t_ms(fn, reps=10):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
    return sorted(ts)[reps // 2]
def pg(dst, st):
    nat.check(lib.gc_hub_pack(x.data_ptr(), K, K, plan.hub_cols.data_ptr(), T, d.data_ptr(), 0, bt.data_ptr(), sc.data_ptr(), st), "p")
    nat.check(lib.gc_hub_gemm(plan.a_hub.data_ptr(), T, a.n_rows, T, bt.data_ptr(), K, 0, sc.data_ptr(), dst.data_ptr(), K, d.data_ptr(), 0, st), "g")
def seq():
    pg(out, torch.cuda.current_stream().cuda_stream)
    sparse._spmm(plan.tail, x, weighted=False, d_row=d, d_col=d, out=out, accumulate=True, relu=True, timer=None)
def conc():
    ev = torch.cuda.Event(); ev.record()
    side.wait_event(ev)
    with torch.cuda.stream(side):
        pg(ch, side.cuda_stream)
        ev2 = torch.cuda.Event(); ev2.record(side)
    sparse._spmm(plan.tail, x, weighted=False, d_row=d, d_col=d, out=out, timer=None)
    torch.cuda.current_stream().wait_event(ev2)
    out.add_(ch).relu_()
r = {"shape": shape, "K": K, "T": T, "seq_ms": t_ms(seq)}
ref = out.clone()
r["conc_ms"] = t_ms(conc)
r["conc_maxdiff"] = float((out - ref).abs().max())
r["plain_ms"] = t_ms(lambda: sparse.spmm_unweighted(a, x, d_col=d, d_row=d, out=out, relu=True))
print(json.dumps(r))
