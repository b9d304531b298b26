#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 python -m pytest -x -q tests/test_gpu_tc_gemm.py tests/test_gpu_parity.py > gpurun_out/w_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/w_tests.log
timeout 300 python tools/gemm_bench.py 2>&1 | grep '"tc"' | cut -c1-140 > gpurun_out/w_gemm.log
MPCG_TC2_SPLIT=0 timeout 300 python tools/gemm_bench.py 2>&1 | grep '"tc"' | cut -c1-140 > gpurun_out/w_gemm_ns.log
MPCG_TC2_TRACE=1 timeout 300 python tools/tc2_trace.py > gpurun_out/w_trace.log 2>&1
