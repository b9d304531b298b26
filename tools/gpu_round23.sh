#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
L=paper_2209_13643_b200/lib
for v in s4c0 s3c0 s3c1 s2c1 s4c1; do
  echo "== $v" >> gpurun_out/var_gemm.log
  MPCG_LIB=$PWD/$L/libmpcg_$v.so timeout 300 python tools/gemm_bench.py 2>&1 | grep '"tc"' | cut -c1-110 >> gpurun_out/var_gemm.log
done
MPCG_LIB=$PWD/$L/libmpcg_s3c1.so timeout 300 python -m pytest -x -q tests/test_gpu_tc_gemm.py > gpurun_out/var_tests.log 2>&1
echo "rc=$?" >> gpurun_out/var_tests.log
