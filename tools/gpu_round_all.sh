#!/bin/bash
# Full round measurement: GPU tests, bench (ours + reference), config table + sweep, GEMM
# micro-bench, dealer split, launch lists and the bench-workload ncu profile.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1200 python -m pytest -q -m gpu tests > gpurun_out/final_tests.log 2>&1; echo "rc=$?" >> gpurun_out/final_tests.log
bash tools/gpu_final_measure.sh
timeout 600 python tools/gemm_bench.py > gpurun_out/gemm_bench.log 2>&1
timeout 1200 python tools/dealer_split.py --out gpurun_out/dealer_split.json > gpurun_out/dealer_split.log 2>&1
MODELS="lenet5 resnet18 vgg16 bert_base" timeout 2400 bash tools/gpu_launches.sh
