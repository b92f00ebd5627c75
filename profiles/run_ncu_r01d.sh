#!/bin/bash
# ncu of the fused GAT aggregation kernels (MODE 1: gathered t_j; MODE 2: SDDMM score)
OUT=gpurun_out/ncu_r01d
mkdir -p $OUT
NCU=/usr/local/cuda/bin/ncu
export GNNC_HUB_HINTS=0 GNNC_SPMM_SHRINK=0   # fixed variant: no autotune launches in the capture
timeout 600 $NCU --set full --clock-control none --import-source on -k regex:spmm_kernel -s 2 -c 1 \
  -o $OUT/gat_reassoc_arxiv_k256 python profiles/gat_probe.py > $OUT/gat1.log 2>&1
timeout 600 $NCU --set full --clock-control none --import-source on -k regex:spmm_kernel -s 5 -c 1 \
  -o $OUT/gat_sddmm_arxiv_k256 python profiles/gat_probe.py > $OUT/gat2.log 2>&1
ls -la $OUT
