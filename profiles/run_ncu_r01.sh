#!/bin/bash
# ncu evidence for the bench workload (run under gpurun; one GPU).
set -x
OUT=gpurun_out/ncu_r01
mkdir -p $OUT
NCU=/usr/local/cuda/bin/ncu
# 1) launch list of the bench command (cold-cache, serialised: compare shares)
timeout 600 $NCU --metrics gpu__time_duration.sum --clock-control none -c 60 --csv \
  --log-file $OUT/launches_reddit_k256.csv python bench.py --steps 2 --warmup 1 --no-sweep --no-cpu > $OUT/launches_run.log 2>&1
# 2) full set on the dominant kernel (SpMM) and the tcgen05 GEMM
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:spmm_kernel -s 2 -c 1 \
  -o $OUT/spmm_reddit_k256 python bench.py --steps 2 --warmup 1 --no-sweep --no-cpu > $OUT/spmm_run.log 2>&1
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:gemm_tf32 -s 2 -c 1 \
  -o $OUT/gemm_reddit_k256 python bench.py --steps 2 --warmup 1 --no-sweep --no-cpu > $OUT/gemm_run.log 2>&1
timeout 600 $NCU --set full --clock-control none --import-source on -k regex:spmm_kernel -s 2 -c 1 \
  -o $OUT/spmm_arxiv_k32 python bench.py --shape arxiv --k 32 --steps 2 --warmup 1 --no-sweep --no-cpu > $OUT/spmm_arxiv_run.log 2>&1
ls -la $OUT
