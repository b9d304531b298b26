# Round-2 (end) profile after the element-by-element chains: ncu launch list of the bench
# command itself, ncu --set full of the register compare chain and of the both-slots GEMM
# inside one ResNet-18 inference, and the BERT-base launch list.
set -u
mkdir -p gpurun_out
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2c_bench_launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu --no-variants --no-blocking > gpurun_out/r2c_bench_under_ncu.log 2>&1
for k in "chain_reg_kernel:5" "ring_gemm_tc3:4"; do
  name=${k%%:*}; cnt=${k##*:}
  MODEL=resnet18 timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
      -k "regex:${name}" -s 0 -c "$cnt" -o "gpurun_out/r2c_${name}" -f python tools/profile_step.py > /dev/null 2>&1
  if [ -f "gpurun_out/r2c_${name}.ncu-rep" ]; then
    ncu -i "gpurun_out/r2c_${name}.ncu-rep" --page raw --csv > "gpurun_out/r2c_${name}_raw.csv" 2>/dev/null
    ncu -i "gpurun_out/r2c_${name}.ncu-rep" --page source --csv > "gpurun_out/r2c_${name}_source.csv" 2>/dev/null
    rm -f "gpurun_out/r2c_${name}.ncu-rep"
  fi
done
MODELS=bert_base bash tools/gpu_launches.sh
ls -la gpurun_out/r2c_*
