#!/bin/bash
# compute-sanitizer over the GPU parity tests on small graphs (kernels run
# ~100x slower under the tool; the GEMM shapes are trimmed):
#  * memcheck over the kernel tests (SpMM / GAT / attention / pack / hub);
#  * memcheck, racecheck (shared-memory hazards) and synccheck (barrier
#    misuse) over the tcgen05 GEMMs: TF32, 3xTF32 (converter warps writing
#    shared memory the MMA reads) and the CTA-pair staircase.
OUT=gpurun_out/sanitizer
mkdir -p $OUT
CS=/usr/local/cuda/bin/compute-sanitizer
GEMM_K="test_gemm and (130-33-16 or 129-7-33 or 700-100-300 or 5-3-7 or 513-256-256)"
timeout 1500 $CS --tool memcheck --error-exitcode 99 --print-limit 20 \
  python -m pytest tests/test_gpu_kernels.py -q -m gpu -x --timeout 1200 \
  -k "not test_gemm[ and not deterministic and not full_size" > $OUT/memcheck_kernels.log 2>&1
echo "memcheck kernels rc=$?" | tee -a $OUT/summary.txt
for tool in memcheck racecheck synccheck; do
  timeout 1200 $CS --tool $tool --error-exitcode 99 --print-limit 20 \
    python -m pytest tests/test_gpu_kernels.py -q -m gpu -x --timeout 1100 \
    -k "$GEMM_K" > $OUT/${tool}_gemm.log 2>&1
  echo "$tool gemm rc=$?" | tee -a $OUT/summary.txt
done
timeout 1500 $CS --tool racecheck --error-exitcode 99 --print-limit 20 \
  python -m pytest tests/test_gpu_kernels.py -q -m gpu -x --timeout 1400 \
  -k "stair_split_matches_oracle and 128 and False" > $OUT/racecheck_stair.log 2>&1
echo "racecheck stair rc=$?" | tee -a $OUT/summary.txt
tail -3 $OUT/*.log
