#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1200 python -m pytest -q -m gpu tests > gpurun_out/r24_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r24_tests.log
timeout 600 python bench.py > gpurun_out/bench.log 2>&1; echo "rc=$?" >> gpurun_out/bench.log
timeout 2400 python tools/run_configs.py --out gpurun_out/configs.json > gpurun_out/run_configs.log 2>&1
timeout 600 python tools/gemm_bench.py > gpurun_out/gemm_bench.log 2>&1
