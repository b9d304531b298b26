#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python tools/run_configs.py --quick --only lenet5,resnet18,vgg16,bert_base --out gpurun_out/configs_quick.json > gpurun_out/run_configs.log 2>&1
MODEL=resnet18 timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:ring_gemm_tc2 -s 1 -c 1 -o gpurun_out/prof_resnet18_tc2 python tools/profile_step.py > /dev/null 2>&1
ncu -i gpurun_out/prof_resnet18_tc2.ncu-rep --page raw --csv > gpurun_out/prof_resnet18_tc2_raw.csv 2>/dev/null
rm -f gpurun_out/prof_resnet18_tc2.ncu-rep
MODEL=bert_base timeout 900 ncu --set full --clock-control none --kernel-name-base demangled -k regex:ring_gemm_tc2 -s 0 -c 6 -o gpurun_out/prof_bert_tc2 python tools/profile_step.py > /dev/null 2>&1
ncu -i gpurun_out/prof_bert_tc2.ncu-rep --page raw --csv > gpurun_out/prof_bert_tc2_raw.csv 2>/dev/null
rm -f gpurun_out/prof_bert_tc2.ncu-rep
