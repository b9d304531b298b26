#!/bin/bash
# Generic A/B measurement on the GPU box: runs the GPU tests, then the given configs under each
# environment assignment in AB (space-separated, e.g. AB="MPCG_TC2_SPLIT=1 MPCG_TC2_SPLIT=0").
#   ONLY=resnet18,vgg16 AB="X=0 X=1" bash tools/gpu_ab.sh
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1200 python -m pytest -x -q -m gpu tests > gpurun_out/ab_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/ab_tests.log
for kv in ${AB:-NONE=1}; do
  env "$kv" timeout 1500 python tools/run_configs.py --only "${ONLY:-resnet18,vgg16,bert_base}" --quick \
      --out "gpurun_out/ab_${kv//=/_}.json" > "gpurun_out/ab_${kv//=/_}.log" 2>&1
done
