# ncu --set full of one SPK level round of a ResNet-18-size ReLU (8.4M elements), SASS source
OUT=${OUT:-adder_l}
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k regex:AdderRound -s 10 -c 1 -o gpurun_out/$OUT -f python tools/relu_probe.py > gpurun_out/${OUT}_ncu.log 2>&1
ncu -i gpurun_out/$OUT.ncu-rep --page raw --csv > gpurun_out/${OUT}_raw.csv 2>/dev/null
ncu -i gpurun_out/$OUT.ncu-rep --page source --csv --print-source sass > gpurun_out/${OUT}_sass.csv 2>/dev/null
rm -f gpurun_out/$OUT.ncu-rep
