#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
MPCG_TC2_SPLIT=1 timeout 600 python -m pytest tests/test_gpu_tc_gemm.py tests/test_gpu_extensions.py -q -x > gpurun_out/pytest_split.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_split.log
for SP in 0 1; do
MPCG_TC2_SPLIT=$SP timeout 900 python tools/run_configs.py --quick --only resnet18,vgg16 --out gpurun_out/cfg_split_$SP.json > gpurun_out/cfg_split_$SP.log 2>&1
done
MPCG_TC2_SPLIT=1 MODEL=resnet18 timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:ring_gemm_tc2 -s 1 -c 1 -o gpurun_out/prof_resnet18_tc2s python tools/profile_step.py > /dev/null 2>&1
ncu -i gpurun_out/prof_resnet18_tc2s.ncu-rep --page raw --csv > gpurun_out/prof_resnet18_tc2s_raw.csv 2>/dev/null
ncu -i gpurun_out/prof_resnet18_tc2s.ncu-rep --page source --csv --print-source sass > gpurun_out/prof_resnet18_tc2s_source.csv 2>/dev/null
rm -f gpurun_out/prof_resnet18_tc2s.ncu-rep
