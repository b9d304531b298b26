#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --no-cpu --no-blocking > gpurun_out/bench.log 2>&1; echo "rc=$?" >> gpurun_out/bench.log
timeout 600 python tools/lenet_knobs.py lenet5 > gpurun_out/knobs_lenet5.log 2>&1
N=$(MODEL=lenet5 python tools/profile_step.py --count 2>/dev/null | tail -1)
MODEL=lenet5 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/lenet5_launches.csv -s "$N" -c "$N" python tools/profile_step.py > /dev/null 2>&1
