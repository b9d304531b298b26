#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:ring_gemm_tc2 -s 1 -c 1 -o gpurun_out/tc2_resnet_merged -f python tools/tc2_trace.py > gpurun_out/ncu_tc2.log 2>&1
ncu -i gpurun_out/tc2_resnet_merged.ncu-rep --page raw --csv > gpurun_out/tc2_resnet_merged_raw.csv 2>/dev/null
ncu -i gpurun_out/tc2_resnet_merged.ncu-rep --page details --csv > gpurun_out/tc2_resnet_merged_details.csv 2>/dev/null
ncu -i gpurun_out/tc2_resnet_merged.ncu-rep --page source --csv > gpurun_out/tc2_resnet_merged_source.csv 2>/dev/null
