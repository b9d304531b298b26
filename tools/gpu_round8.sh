#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python tools/run_configs.py --quick --only resnet18,vgg16,lenet5 --out gpurun_out/configs_quick.json > gpurun_out/run_configs.log 2>&1
MPCG_TC2_PACKL=1 timeout 900 python tools/run_configs.py --quick --only resnet18,vgg16 --out gpurun_out/configs_quick_packl.json > gpurun_out/run_configs_packl.log 2>&1
for M in resnet18 lenet5; do
N=$(MODEL=$M python tools/profile_step.py --count 2>/dev/null | tail -1)
MODEL=$M timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${M}_launches.csv -s "$N" -c "$N" python tools/profile_step.py > /dev/null 2>&1
done
MODEL=resnet18 timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:ring_gemm_tc2 -s 1 -c 1 -o gpurun_out/prof_resnet18_tc2 python tools/profile_step.py > /dev/null 2>&1
ncu -i gpurun_out/prof_resnet18_tc2.ncu-rep --page raw --csv > gpurun_out/prof_resnet18_tc2_raw.csv 2>/dev/null
ncu -i gpurun_out/prof_resnet18_tc2.ncu-rep --page source --csv --print-source sass > gpurun_out/prof_resnet18_tc2_source.csv 2>/dev/null
rm -f gpurun_out/prof_resnet18_tc2.ncu-rep
