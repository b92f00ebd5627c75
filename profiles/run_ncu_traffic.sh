#!/bin/bash
# DRAM traffic of the dominant kernel (SpMM) per composition for the bench
# workload (Reddit-shaped, K = 256): one ncu capture per composition.
OUT=gpurun_out/ncu_traffic
mkdir -p $OUT
NCU=/usr/local/cuda/bin/ncu
for comp in precompute:aggregate_first precompute:update_first dynamic:aggregate_first dynamic:update_first; do
  tag=${comp/:/_}
  timeout 600 $NCU --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct,lts__throughput.avg.pct_of_peak_sustained_elapsed \
    --clock-control none -k regex:spmm_kernel -s 2 -c 1 --csv --log-file $OUT/$tag.csv \
    python bench.py --steps 2 --warmup 1 --no-sweep --no-cpu --no-extra --composition $comp > $OUT/$tag.log 2>&1
done
ls -la $OUT
