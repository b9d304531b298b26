#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 python tools/lenet_knobs.py lenet5 > gpurun_out/knobs_lenet5.log 2>&1
for M in resnet18 vgg16; do
  N=$(MODEL=$M python tools/profile_step.py --count 2>/dev/null | tail -1)
  MODEL=$M timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${M}_launches.csv -s "$N" -c "$N" python tools/profile_step.py > /dev/null 2>&1
  MODEL=$M timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:ring_gemm_tc2 -s 0 -c 6 -o gpurun_out/prof_${M}_tc2 python tools/profile_step.py > /dev/null 2>&1
  ncu -i gpurun_out/prof_${M}_tc2.ncu-rep --page raw --csv > gpurun_out/prof_${M}_tc2_raw.csv 2>/dev/null
  ncu -i gpurun_out/prof_${M}_tc2.ncu-rep --page source --csv --print-source sass > gpurun_out/prof_${M}_tc2_source.csv 2>/dev/null
  rm -f gpurun_out/prof_${M}_tc2.ncu-rep
done
