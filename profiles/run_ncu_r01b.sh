#!/bin/bash
# ncu evidence for the bench workload after the SpMM rework (run under gpurun; one GPU).
OUT=gpurun_out/ncu_r01b
mkdir -p $OUT
NCU=/usr/local/cuda/bin/ncu
KRE='regex:spmm_kernel|spmm_fixup|gemm_tf32|gemm_fp32|transpose_kernel|sddmm|softmax|node_proj|scale_rows'
# launch list of our kernels in the bench command (cold-cache, serialised: compare SHARES)
timeout 600 $NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k "$KRE" -c 40 --csv \
  --log-file $OUT/launches_reddit_k256.csv python bench.py --steps 2 --warmup 1 --no-sweep --no-cpu --no-extra > $OUT/launches_run.log 2>&1
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:spmm_kernel -s 2 -c 1 \
  -o $OUT/spmm_reddit_k256 python bench.py --steps 2 --warmup 1 --no-sweep --no-cpu --no-extra > $OUT/spmm_run.log 2>&1
timeout 600 $NCU --set full --clock-control none --import-source on -k regex:spmm_kernel -s 2 -c 1 \
  -o $OUT/spmm_arxiv_k32 python bench.py --shape arxiv --k 32 --steps 2 --warmup 1 --no-sweep --no-cpu --no-extra > $OUT/spmm_arxiv_run.log 2>&1
ls -la $OUT
