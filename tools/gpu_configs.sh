#!/bin/bash
# Per-config end-to-end runs on one B200 (both parties on cuda:0): writes gpurun_out/cfg_*.json
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for spec in "mlp:--check" "lenet5:--check" "toy_cnn:--check" "toy_transformer:--check" "vgg16:--check" "vgg16:--link 10gbps --iters 1"; do
  m=${spec%%:*}; args=${spec#*:}
  tag=$(echo "$m $args" | tr -c 'a-z0-9' '_')
  timeout 900 python tools/run_model.py $m $args > gpurun_out/cfg_${tag}.log 2>&1
  echo "$m $args rc=$?" >> gpurun_out/cfg_status.txt
done
