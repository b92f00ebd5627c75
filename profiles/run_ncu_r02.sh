#!/bin/bash
# Round-2 ncu evidence.  (1) the bench line, then ncu of the SAME
# configuration (split and composition the bench's autotuner/selector chose,
# forced for the profiled runs): per-launch list with DRAM bytes and full
# sections of the tail SpMM and the staircase GEMM; (2) every GAT-path kernel
# on arxiv (1 and 4 heads, K = 32/256/1024) and the products SpMM.
OUT=${OUT:-gpurun_out/ncu_r02}
mkdir -p $OUT
NCU=/usr/local/cuda/bin/ncu
timeout 1500 python bench.py --out $OUT/bench.json > $OUT/bench.log 2>&1
SPLIT=$(python -c "import json; print(json.load(open('$OUT/bench.json'))['dense_split']['chosen'])")
COMP=$(python -c "import json; print(json.load(open('$OUT/bench.json'))['config']['composition'])")
echo "forcing split=$SPLIT composition=$COMP" > $OUT/forced.txt
export GNNC_HUB_HINTS=0 GNNC_SPMM_SHRINK=0 GNNC_HUB_SPLIT=$SPLIT
B="python bench.py --steps 2 --warmup 3 --no-sweep --no-cpu --no-extra --no-fp32-class --parity-rows 8 --composition $COMP"
timeout 900 $NCU --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  --clock-control none --csv --log-file $OUT/launches.csv $B > $OUT/launches_run.log 2>&1
timeout 900 $NCU --profile-from-start off --set full --clock-control none --import-source on -k regex:spmm_kernel -c 1 \
  -o $OUT/spmm_tail_reddit_k256 $B > $OUT/spmm_run.log 2>&1
timeout 900 $NCU --profile-from-start off --set full --clock-control none --import-source on -k regex:gemm_hub_pair -c 1 \
  -o $OUT/hub_gemm_reddit_k256 $B > $OUT/hub_run.log 2>&1
unset GNNC_HUB_SPLIT
timeout 900 python profiles/probes/gat_ncu.py --products > $OUT/gat_probe.json 2>$OUT/gat_probe.err
timeout 1500 $NCU --profile-from-start off --set full --clock-control none -o $OUT/gat_path \
  python profiles/probes/gat_ncu.py --products > $OUT/gat_run.log 2>&1
ls -la $OUT
