# round-2 measurement pass: GPU tests, bench line (ours + reference arm), ncu launch list of the
# bench command, ncu --set full of the dominant kernels of the bench workload (ResNet-18)
set -u
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q 2>&1 | tail -15 > gpurun_out/r2p_pytest.txt
timeout 900 python bench.py > gpurun_out/r2p_bench.json 2> gpurun_out/r2p_bench.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r2p_bench_ref.json 2> gpurun_out/r2p_bench_ref.err
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2p_bench_launches.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu --no-variants --no-blocking > gpurun_out/r2p_bench_under_ncu.log 2>&1
for k in "AdderRound:6" "ring_gemm_tc2:6" "EpsIm2col:2" "ChainStep:4"; do
  name=${k%%:*}; cnt=${k##*:}
  MODEL=resnet18 timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
      -k "regex:${name}" -s 0 -c "$cnt" -o "gpurun_out/r2p_${name}" -f python tools/profile_step.py > /dev/null 2>&1
  if [ -f "gpurun_out/r2p_${name}.ncu-rep" ]; then
    ncu -i "gpurun_out/r2p_${name}.ncu-rep" --page raw --csv > "gpurun_out/r2p_${name}_raw.csv" 2>/dev/null
    rm -f "gpurun_out/r2p_${name}.ncu-rep"
  fi
done
tail -3 gpurun_out/r2p_pytest.txt; cut -c1-300 gpurun_out/r2p_bench.json; cut -c1-300 gpurun_out/r2p_bench_ref.json; ls -la gpurun_out | tail -20
