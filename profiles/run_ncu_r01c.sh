#!/bin/bash
# ncu: persistent tcgen05 GEMM and the fused GAT aggregation (one GPU).
OUT=gpurun_out/ncu_r01c
mkdir -p $OUT
NCU=/usr/local/cuda/bin/ncu
cat > /tmp/gemm_probe.py <<'PY'
import sys, torch
sys.path.insert(0, ".")
import paper_2306_15155_b200 as gc
dev = torch.device("cuda", 0)
for (M, K, N) in ((232965, 256, 256), (169343, 1024, 1024), (2449029, 256, 256)):
    a = torch.rand(M, K, device=dev) - 0.5
    w = torch.rand(K, N, device=dev) - 0.5
    for _ in range(3):
        gc.gemm(a, w)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        gc.gemm(a, w)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    print(f"gemm M={M} K={K} N={N}: {ms:.4f} ms  {2*M*K*N/ms/1e9:.1f} TFLOP/s  {4*(M*K+K*N+M*N)/ms/1e6:.1f} GB/s", flush=True)
PY
timeout 300 python /tmp/gemm_probe.py > $OUT/gemm_probe.txt 2>&1
cat $OUT/gemm_probe.txt
timeout 600 $NCU --set full --clock-control none --import-source on -k regex:gemm_tf32 -s 13 -c 1 \
  -o $OUT/gemm_tf32_k1024 python /tmp/gemm_probe.py > $OUT/gemm_ncu_run.log 2>&1
timeout 600 $NCU --set full --clock-control none --import-source on -k regex:spmm_kernel -s 4 -c 1 \
  -o $OUT/gat_fused_arxiv_k256 python bench.py --shape arxiv --k 256 --steps 2 --warmup 1 --no-sweep --no-cpu --no-extra --composition precompute:aggregate_first > $OUT/gat_run.log 2>&1
ls -la $OUT
