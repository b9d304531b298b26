#!/bin/bash
# Launch lists (ncu gpu__time_duration only; cold-cache, serialised) of one eager inference
# per model: gpurun_out/<model>_launches.csv
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for M in ${MODELS:-lenet5 resnet18 vgg16 bert_base}; do
  N=$(MODEL=$M python tools/profile_step.py --count 2>/dev/null | tail -1)
  MODEL=$M timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${M}_launches.csv \
      -s "$N" -c "$N" python tools/profile_step.py > /dev/null 2>&1
done
