"""Dense update H·W in the three numerics modes (TF32, 3xTF32 = the fp32
class, exact SIMT) at the BASELINE shapes: CUDA-event ms, TFLOP/s, HBM GB/s."""
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import paper_2306_15155_b200 as gc  # noqa: E402

dev = torch.device("cuda", 0)
res = []
for (M, K, N, name) in [(232965, 256, 256, "reddit K=256"), (232965, 32, 32, "reddit K=32"),
                        (232965, 1024, 1024, "reddit K=1024"), (169343, 1024, 1024, "arxiv K=1024"),
                        (2449029, 256, 256, "products K=256"), (2708, 1433, 16, "cora L1"),
                        (65536, 8192, 8192, "compute-bound (TF32 peak probe)")]:
    a = torch.rand(M, K, device=dev) - 0.5
    w = torch.rand(K, N, device=dev) - 0.5
    ref = (a.double() @ w.double()) if M * K * N < 2 ** 40 else None
    row = {"shape": name, "M": M, "K": K, "N": N}
    for prec in ("tf32", "fp32", "simt"):
        out = gc.gemm(a, w, precision=prec)
        err = float((out.double() - ref).abs().max() / ref.abs().max()) if ref is not None else None
        if prec == "simt" and ref is None:
            continue
        for _ in range(3):
            gc.gemm(a, w, precision=prec, out=out)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        reps = 10
        for _ in range(reps):
            gc.gemm(a, w, precision=prec, out=out)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        row[prec] = {"ms": round(ms, 4), "tflops": round(2 * M * K * N / ms / 1e9, 1),
                     "gbs": round(4 * (M * K + K * N + M * N) / ms / 1e6, 1), "maxrel": err}
    res.append(row)
    print(json.dumps(row), flush=True)
    del a, w, ref, out
    torch.cuda.empty_cache()
Path("gpurun_out").mkdir(exist_ok=True)
Path("gpurun_out/gemm_modes.json").write_text(json.dumps(res, indent=1))
