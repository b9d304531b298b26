#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for cfg in "1 0" "1 1" "1 2" "1 3" "1 5" "0 3"; do
  set -- $cfg
  echo "SPLIT=$1 L2AHEAD=$2" >> gpurun_out/pf_gemm.log
  MPCG_TC2_SPLIT=$1 MPCG_TC2_L2AHEAD=$2 timeout 300 python tools/gemm_bench.py 2>&1 | grep '"tc"' | cut -c1-120 >> gpurun_out/pf_gemm.log
done
MPCG_TC2_TRACE=1 timeout 300 python tools/tc2_trace.py > gpurun_out/pf_trace.log 2>&1
