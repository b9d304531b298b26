#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python tools/run_configs.py --quick --only bert_base,resnet18,vgg16,lenet5,mlp --out gpurun_out/configs_quick.json > gpurun_out/run_configs.log 2>&1
N=$(MODEL=bert_base python tools/profile_step.py --count 2>/dev/null | tail -1)
MODEL=bert_base timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/bert_base_launches.csv -s "$N" -c "$N" python tools/profile_step.py > /dev/null 2>&1
