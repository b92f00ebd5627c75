#!/bin/bash
# compute-sanitizer memcheck over the GPU parity tests on small graphs
# (kernels run ~100x slower under the tool; the GEMM shapes are trimmed).
OUT=gpurun_out/sanitizer
mkdir -p $OUT
CS=/usr/local/cuda/bin/compute-sanitizer
timeout 1500 $CS --tool memcheck --error-exitcode 99 --print-limit 20 \
  python -m pytest tests/test_gpu_kernels.py -q -m gpu -x --timeout 1200 \
  -k "not test_gemm[ and not multihead and not deterministic" > $OUT/memcheck_kernels.log 2>&1
echo "memcheck kernels rc=$?" | tee -a $OUT/summary.txt
timeout 900 $CS --tool memcheck --error-exitcode 99 --print-limit 20 \
  python -m pytest tests/test_gpu_kernels.py -q -m gpu -x --timeout 800 \
  -k "test_gemm and (130-33-16 or 129-7-33 or 700-100-300 or 5-3-7)" > $OUT/memcheck_gemm.log 2>&1
echo "memcheck gemm rc=$?" | tee -a $OUT/summary.txt
tail -3 $OUT/memcheck_kernels.log $OUT/memcheck_gemm.log
