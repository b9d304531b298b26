#!/bin/bash
# compute-sanitizer memcheck over a subset of the GPU tests (small shapes): out-of-bounds and
# misaligned device accesses, invalid frees, leaked device allocations at exit.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
export MPCG_SLOW_TESTS=0
for T in "tests/test_gpu_parity.py" "tests/test_gpu_tc_gemm.py" "tests/test_gpu_fused_opens.py" "tests/test_gpu_extensions.py"; do
  n=$(basename $T .py)
  timeout 1500 compute-sanitizer --tool memcheck --print-limit 20 --error-exitcode 97 \
      python -m pytest -x -q -m gpu "$T" > gpurun_out/sanitize_$n.log 2>&1
  echo "rc=$?" >> gpurun_out/sanitize_$n.log
done
