#!/bin/bash
cd /root/repo
MODEL=${MODEL:-resnet18} timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:${KREGEX:-EpsIm2colPair} -s ${KSKIP:-1} -c 1 -o gpurun_out/${OUT:-eps_resnet} -f python tools/profile_step.py > gpurun_out/ncu_eps.log 2>&1
ncu -i gpurun_out/${OUT:-eps_resnet}.ncu-rep --page details --csv > gpurun_out/${OUT:-eps_resnet}_details.csv 2>/dev/null
ncu -i gpurun_out/${OUT:-eps_resnet}.ncu-rep --page source --csv > gpurun_out/${OUT:-eps_resnet}_source.csv 2>/dev/null
rm -f gpurun_out/${OUT:-eps_resnet}.ncu-rep
