#!/bin/bash
# Round-1 refresh (current kernels): launch list of the bench's timed region
# (cudaProfilerStart/Stop bracket it; --profile-from-start off), then one
# --set full capture of the SpMM and of the GEMM inside that region.
OUT=gpurun_out/ncu_r01e
mkdir -p $OUT
NCU=/usr/local/cuda/bin/ncu
export GNNC_HUB_HINTS=0 GNNC_SPMM_SHRINK=0   # fixed variant: no autotune launches in the captures
B="python bench.py --steps 2 --warmup 3 --no-sweep --no-cpu --no-extra"
timeout 900 $NCU --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  --clock-control none --csv --log-file $OUT/launches.csv $B > $OUT/launches_run.log 2>&1
timeout 900 $NCU --profile-from-start off --set full --clock-control none --import-source on -k regex:spmm_kernel -c 1 \
  -o $OUT/spmm_reddit_k256 $B > $OUT/spmm_run.log 2>&1
timeout 900 $NCU --profile-from-start off --set full --clock-control none --import-source on -k regex:gemm -c 1 \
  -o $OUT/gemm_reddit_k256 $B > $OUT/gemm_run.log 2>&1
ls -la $OUT
