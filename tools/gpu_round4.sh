#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_tc_gemm.py -x -q > gpurun_out/pytest_tc.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_tc.log
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
timeout 1800 python tools/run_configs.py --quick > gpurun_out/run_configs.log 2>&1; echo "rc=$?" >> gpurun_out/run_configs.log
timeout 600 python bench.py --no-cpu > gpurun_out/bench.log 2>&1; echo "rc=$?" >> gpurun_out/bench.log
MODEL=resnet18 timeout 600 ncu --set full --clock-control none --import-source on -k regex:ring_gemm_tc2 -s 2 -c 1 -o gpurun_out/prof_tc2_resnet python tools/profile_step.py > /dev/null 2>&1
ncu -i gpurun_out/prof_tc2_resnet.ncu-rep --page raw --csv > gpurun_out/prof_tc2_resnet_raw.csv 2>/dev/null
rm -f gpurun_out/prof_tc2_resnet.ncu-rep
