#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1200 python -m pytest -x -q -m gpu tests > gpurun_out/o_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/o_tests.log
timeout 600 python bench.py > gpurun_out/o_bench.log 2>&1
timeout 900 python tools/run_configs.py --only resnet18,vgg16,bert_base,lenet5,mlp --quick --out gpurun_out/o_configs.json > gpurun_out/o_configs.log 2>&1
