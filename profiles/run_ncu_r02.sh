#!/bin/bash
# Round-2 ncu evidence.  (1) a short bench line (the composition and dense
# split the selector / autotuner pick), then ncu of the SAME configuration
# (forced for the profiled runs): per-launch list with DRAM bytes and full
# sections of the tail SpMM and the staircase GEMM; (2) every GAT-path kernel
# on arxiv (1 and 4 heads, K = 32/256/1024) and the products SpMM.  Reports
# are reduced to CSV + a markdown summary on the box (gpurun copies back at
# most 64 MiB).
OUT=${OUT:-gpurun_out/ncu_r02}
mkdir -p $OUT
NCU=/usr/local/cuda/bin/ncu
timeout 900 python bench.py --no-sweep --no-extra --no-cpu --no-fp32-class --out $OUT/bench_short.json > $OUT/bench.log 2>&1
SPLIT=$(python -c "import json; print(json.load(open('$OUT/bench_short.json'))['dense_split']['chosen'])")
COMP=$(python -c "import json; print(json.load(open('$OUT/bench_short.json'))['config']['composition'])")
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
timeout 1500 $NCU --profile-from-start off --set full --clock-control none \
  -k "regex:spmm_kernel|edge_softmax|attn_score|node_proj|pack_rows" -o $OUT/gat_path \
  python profiles/probes/gat_ncu.py --products > $OUT/gat_run.log 2>&1
for r in $OUT/*.ncu-rep; do $NCU -i $r --page raw --csv > ${r%.ncu-rep}.raw.csv 2>/dev/null; done
python profiles/summarize_ncu.py $OUT/*.ncu-rep > $OUT/summary.md 2>$OUT/summary.err
rm -f $OUT/gat_path.ncu-rep
gzip -f $OUT/*.raw.csv
du -sh $OUT; ls -la $OUT
