#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1200 python -m pytest -x -q -m gpu tests > gpurun_out/f_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/f_tests.log
MPCG_EPS_FUSE=0 timeout 900 python tools/run_configs.py --only resnet18,vgg16,bert_base --quick --out gpurun_out/f0_configs.json > gpurun_out/f0_configs.log 2>&1
timeout 900 python tools/run_configs.py --only resnet18,vgg16,bert_base,lenet5,mlp --quick --out gpurun_out/f1_configs.json > gpurun_out/f1_configs.log 2>&1
MPCG_TC2_TRACE=1 timeout 300 python tools/tc2_trace.py > gpurun_out/f_trace.log 2>&1
