# ncu --set full of one ring-GEMM kernel launch (KREGEX, default the both-slots kernel) at one
# shape, raw + SASS source pages exported as CSV.
M=${M:-131072}; K=${K:-576}; N=${N:-64}; OUT=${OUT:-tc3_l1}; KREGEX=${KREGEX:-ring_gemm_tc3}
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k regex:$KREGEX -s 1 -c 1 -o gpurun_out/$OUT -f python ${PROBE:-tools/tc3_bench.py ${M}x${K}x${N}} > gpurun_out/${OUT}_ncu.log 2>&1
ncu -i gpurun_out/$OUT.ncu-rep --page raw --csv > gpurun_out/${OUT}_raw.csv 2>/dev/null
ncu -i gpurun_out/$OUT.ncu-rep --page source --csv --print-source sass > gpurun_out/${OUT}_sass.csv 2>/dev/null
rm -f gpurun_out/$OUT.ncu-rep
