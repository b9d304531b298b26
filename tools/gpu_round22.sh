#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 python -m pytest -x -q tests/test_gpu_tc_gemm.py tests/test_gpu_parity.py > gpurun_out/coal_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/coal_tests.log
timeout 300 python tools/gemm_bench.py 2>&1 | grep '"tc"' | cut -c1-140 > gpurun_out/coal_gemm.log
MPCG_TC2_TRACE=1 timeout 300 python tools/tc2_trace.py > gpurun_out/coal_trace.log 2>&1
timeout 900 python tools/run_configs.py --only resnet18,vgg16 --quick --out gpurun_out/coal_configs.json > gpurun_out/coal_configs.log 2>&1
