#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for sp in 1 0; do
  echo "SPLIT=$sp" >> gpurun_out/s_gemm.log
  MPCG_TC2_SPLIT=$sp timeout 300 python tools/gemm_bench.py 2>&1 | grep '"tc"' | cut -c1-100 >> gpurun_out/s_gemm.log
done
MPCG_TC2_SPLIT=0 timeout 900 python tools/run_configs.py --only resnet18,vgg16 --quick --out gpurun_out/s0_configs.json > gpurun_out/s0_configs.log 2>&1
