#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 python -m pytest -x -q tests/test_gpu_tc_gemm.py > gpurun_out/at_tests.log 2>&1
echo "tests AT0 rc=$?" >> gpurun_out/at_tests.log
MPCG_TC2_AT=1 timeout 600 python -m pytest -x -q tests/test_gpu_tc_gemm.py >> gpurun_out/at_tests.log 2>&1
echo "tests AT1 rc=$?" >> gpurun_out/at_tests.log
MPCG_TC2_TRACE=1 timeout 300 python tools/tc2_trace.py > gpurun_out/at0_trace.log 2>&1
MPCG_TC2_AT=1 MPCG_TC2_TRACE=1 timeout 300 python tools/tc2_trace.py > gpurun_out/at_trace.log 2>&1
MPCG_TC2_TRACE=1 timeout 300 python tools/tc2_trace.py 1024 768 3072 > gpurun_out/at0_trace_bert.log 2>&1
MPCG_TC2_AT=0 timeout 600 python tools/gemm_bench.py > gpurun_out/at0_gemm.log 2>&1
MPCG_TC2_AT=1 timeout 600 python tools/gemm_bench.py > gpurun_out/at1_gemm.log 2>&1
MPCG_TC2_AT=0 timeout 900 python tools/run_configs.py --only resnet18,vgg16,bert_base --quick --out gpurun_out/at0_configs.json > gpurun_out/at0_configs.log 2>&1
MPCG_TC2_AT=1 timeout 900 python tools/run_configs.py --only resnet18,vgg16 --quick --out gpurun_out/at1_configs.json > gpurun_out/at1_configs.log 2>&1
