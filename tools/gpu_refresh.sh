#!/bin/bash
# End-of-round refresh: bench line (ours + reference arm) and the full config table + sweep.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 python bench.py > gpurun_out/bench.log 2>&1; echo "rc=$?" >> gpurun_out/bench.log
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.log 2>&1
timeout 2400 python tools/run_configs.py --out gpurun_out/configs.json > gpurun_out/run_configs.log 2>&1
