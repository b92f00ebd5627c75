#!/bin/bash
# Round-1 (hub split, CTA-pair hub GEMM): full bench line, the launch list of the bench's timed
# region (--profile-from-start off; cudaProfilerStart/Stop bracket it), and one
# --set full capture each of the tail SpMM and the hub GEMM inside it.
OUT=gpurun_out/ncu_r01k
mkdir -p $OUT
NCU=/usr/local/cuda/bin/ncu
timeout 1500 python bench.py --out $OUT/bench.json > $OUT/bench.log 2>&1
export GNNC_HUB_HINTS=0 GNNC_SPMM_SHRINK=0   # fixed SpMM variant: no autotune launches in the captures
B="python bench.py --steps 2 --warmup 3 --no-sweep --no-cpu --no-extra"
timeout 900 $NCU --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  --clock-control none --csv --log-file $OUT/launches.csv $B > $OUT/launches_run.log 2>&1
timeout 900 $NCU --profile-from-start off --set full --clock-control none --import-source on -k regex:spmm_kernel -c 1 \
  -o $OUT/spmm_tail_reddit_k256 $B > $OUT/spmm_run.log 2>&1
timeout 900 $NCU --profile-from-start off --set full --clock-control none --import-source on -k regex:gemm_hub_pair -c 1 \
  -o $OUT/hub_gemm_reddit_k256 $B > $OUT/hub_run.log 2>&1
timeout 900 $NCU --profile-from-start off --set full --clock-control none --import-source on -k regex:gemm_tf32 -c 1 \
  -o $OUT/gemm_tf32_reddit_k256 $B > $OUT/gemm_run.log 2>&1
ls -la $OUT
