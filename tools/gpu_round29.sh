#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1200 python -m pytest -x -q -m gpu tests > gpurun_out/g_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/g_tests.log
timeout 300 python tools/gemm_bench.py 2>&1 | grep '"tc"' | cut -c1-100 > gpurun_out/g_gemm.log
MPCG_TC2_TRACE=1 timeout 300 python tools/tc2_trace.py > gpurun_out/g_trace.log 2>&1
timeout 900 python tools/run_configs.py --only resnet18,vgg16,bert_base --quick --out gpurun_out/g_configs.json > gpurun_out/g_configs.log 2>&1
