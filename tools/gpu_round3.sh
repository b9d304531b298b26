#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_tc_gemm.py -x -q > gpurun_out/pytest_tc.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_tc.log
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python tools/run_model.py vgg16 --mode blocking --iters 3 > gpurun_out/cfg_vgg16.log 2>&1; echo "rc=$?" >> gpurun_out/cfg_vgg16.log
timeout 900 python tools/run_model.py resnet18 --check --mode blocking --iters 2 --no-graph > gpurun_out/cfg_resnet18.log 2>&1; echo "rc=$?" >> gpurun_out/cfg_resnet18.log
timeout 900 python tools/run_model.py bert_base --check --mode blocking --iters 1 --no-graph > gpurun_out/cfg_bert_base.log 2>&1; echo "rc=$?" >> gpurun_out/cfg_bert_base.log
timeout 600 python bench.py --no-cpu > gpurun_out/bench.log 2>&1; echo "rc=$?" >> gpurun_out/bench.log
N=$(MODEL=resnet18 python tools/profile_step.py --count 2>/dev/null | tail -1)
MODEL=resnet18 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/resnet_launches.csv -s "$N" -c "$N" python tools/profile_step.py > /dev/null 2>&1
MODEL=resnet18 timeout 600 ncu --set full --clock-control none --import-source on -k regex:ring_gemm_tc2 -s 2 -c 1 -o gpurun_out/prof_tc2_resnet python tools/profile_step.py > /dev/null 2>&1
ncu -i gpurun_out/prof_tc2_resnet.ncu-rep --page raw --csv > gpurun_out/prof_tc2_resnet_raw.csv 2>/dev/null
ncu -i gpurun_out/prof_tc2_resnet.ncu-rep --page source --csv --print-source sass > gpurun_out/prof_tc2_resnet_source.csv 2>/dev/null
rm -f gpurun_out/prof_tc2_resnet.ncu-rep
