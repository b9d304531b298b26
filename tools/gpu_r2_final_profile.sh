# Round-2 profile of the bench workload (ResNet-18 b128 pipelined): ncu launch list of the bench
# command itself, and ncu --set full of the two dominant kernel classes inside one inference.
set -u
mkdir -p gpurun_out
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2f_bench_launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu --no-variants --no-blocking > gpurun_out/r2f_bench_under_ncu.log 2>&1
for k in "ring_gemm_tc3:4" "AdderRound:6"; do
  name=${k%%:*}; cnt=${k##*:}
  MODEL=resnet18 timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
      -k "regex:${name}" -s 0 -c "$cnt" -o "gpurun_out/r2f_${name}" -f python tools/profile_step.py > /dev/null 2>&1
  if [ -f "gpurun_out/r2f_${name}.ncu-rep" ]; then
    ncu -i "gpurun_out/r2f_${name}.ncu-rep" --page raw --csv > "gpurun_out/r2f_${name}_raw.csv" 2>/dev/null
    rm -f "gpurun_out/r2f_${name}.ncu-rep"
  fi
done
ls -la gpurun_out/r2f_*
