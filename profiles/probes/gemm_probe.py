"""TF32 GEMM H·W timings on the benchmark shapes (GNNC_GEMM_PAIR=0|1)."""
import sys, os, json
import torch
sys.path.insert(0, ".")
import paper_2306_15155_b200 as gc
dev = torch.device("cuda", 0)
res = {"pair": os.environ.get("GNNC_GEMM_PAIR", "1")}
for (M, K, N) in ((232965, 256, 256), (169343, 1024, 1024), (232965, 1024, 1024), (2449029, 256, 256),
                  (169343, 256, 1024)):
    a = torch.rand(M, K, device=dev) - 0.5
    w = torch.rand(K, N, device=dev) - 0.5
    for _ in range(3): gc.gemm(a, w)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10): out = gc.gemm(a, w)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    ref = (a[:512].double() @ w.double())
    err = float((out[:512].double() - ref).abs().max() / ref.abs().max())
    res[f"{M}x{K}x{N}"] = {"ms": round(ms, 4), "tflops": round(2 * M * K * N / ms / 1e9, 1),
                           "hbm_gbs": round(4 * (M * K + K * N + M * N) / ms / 1e6, 1), "rel_err": err}
    del a, w, out
print(json.dumps(res))
