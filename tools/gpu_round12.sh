#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for L in 0 3 8; do
MPCG_TC2_L2AHEAD=$L timeout 600 python tools/run_configs.py --quick --only resnet18 --out gpurun_out/cfg_l2_$L.json > gpurun_out/cfg_l2_$L.log 2>&1
done
timeout 600 python bench.py --no-cpu --no-blocking > gpurun_out/bench.log 2>&1
N=$(MODEL=resnet18 python tools/profile_step.py --count 2>/dev/null | tail -1)
MODEL=resnet18 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/resnet18_launches.csv -s "$N" -c "$N" python tools/profile_step.py > /dev/null 2>&1
