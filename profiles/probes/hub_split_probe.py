"""Probe: split Ã's columns into T hub columns (dense, tensor cores) + a
sparse tail (SpMM).  Times the tail SpMM and a torch bf16 GEMM proxy for the
hub block (3-term bf16 split of the gathered operand) on the Reddit shape."""
import sys, time, json
import torch
sys.path.insert(0, ".")
import paper_2306_15155_b200 as gc
from paper_2306_15155_b200 import graphs, sparse
from paper_2306_15155_b200.sparse import CsrMatrix

dev = torch.device("cuda", 0)
torch.cuda.set_device(dev)
shape = sys.argv[1] if len(sys.argv) > 1 else "reddit"
a = graphs.shape_graph(shape, device=dev)
a = sparse.add_self_loops(a)
n = a.n_rows
K = int(sys.argv[2]) if len(sys.argv) > 2 else 256
h = torch.rand(n, K, device=dev) - 0.5
d = sparse.inv_sqrt_degrees(a).to(dev)

def t_ms(fn, reps=10):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(reps):
        e0.record(); fn(); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
    ts.sort(); return ts[len(ts)//2]

res = {"shape": shape, "K": K, "n": n, "m": a.nnz}
res["full_spmm_ms"] = t_ms(lambda: sparse.spmm_unweighted(a, h, d_col=d, d_row=d))
deg = torch.bincount(a.col_idx.long(), minlength=a.n_cols)
order = torch.argsort(deg, descending=True)
for T in (512, 1024, 2048, 4096, 8192):
    hub = torch.zeros(a.n_cols, dtype=torch.bool, device=dev); hub[order[:T]] = True
    keep = ~hub[a.col_idx.long()]
    rows = torch.repeat_interleave(torch.arange(n, device=dev), a.row_ptr[1:].long() - a.row_ptr[:-1].long())
    cnt = torch.bincount(rows[keep], minlength=n)
    rp = torch.zeros(n + 1, dtype=torch.int32, device=dev); rp[1:] = torch.cumsum(cnt, 0).int()
    tail = CsrMatrix(n, a.n_cols, rp, a.col_idx[keep].contiguous(), torch.ones(int(keep.sum()), device=dev), validate=False)
    t_tail = t_ms(lambda: sparse.spmm_unweighted(tail, h, d_col=d, d_row=d))
    A = torch.zeros(n, T, dtype=torch.bfloat16, device=dev)
    pos = torch.full((a.n_cols,), -1, dtype=torch.long, device=dev); pos[order[:T]] = torch.arange(T, device=dev)
    hr = rows[~keep]; hc = pos[a.col_idx.long()[~keep]]
    A[hr, hc] = 1
    B3 = torch.randn(3 * T, K, device=dev).to(torch.bfloat16)
    A3 = torch.cat([A, A, A], 1)
    t_g3 = t_ms(lambda: A3 @ B3)
    B1 = torch.randn(T, 3 * K, device=dev).to(torch.bfloat16)
    t_g1 = t_ms(lambda: A @ B1)
    res[f"T{T}"] = {"hub_edges_frac": 1 - tail.nnz / a.nnz, "tail_ms": t_tail, "gemm3k_ms": t_g1, "gemm3T_ms": t_g3}
    print(json.dumps(res[f"T{T}"]), flush=True)
    del A, A3, B3, B1, tail
print(json.dumps(res))
