# ncu --set full of one tcgen05 ring GEMM (ResNet-18 layer1 conv shape by default) with the
# source page (SASS + stall reasons) exported as CSV for reading here.
M=${M:-131072}; K=${K:-576}; N=${N:-64}; OUT=${OUT:-tc2_l1}
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k regex:ring_gemm_tc2 -s 1 -c 1 -o gpurun_out/$OUT -f python tools/tc2_trace.py $M $K $N > gpurun_out/${OUT}_ncu.log 2>&1
ncu -i gpurun_out/$OUT.ncu-rep --page raw --csv > gpurun_out/${OUT}_raw.csv 2>/dev/null
ncu -i gpurun_out/$OUT.ncu-rep --page source --csv --print-source sass > gpurun_out/${OUT}_sass.csv 2>/dev/null
ncu -i gpurun_out/$OUT.ncu-rep --page details --csv > gpurun_out/${OUT}_details.csv 2>/dev/null
rm -f gpurun_out/$OUT.ncu-rep
ls -la gpurun_out/${OUT}_*
