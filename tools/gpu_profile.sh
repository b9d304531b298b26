#!/bin/bash
# Profiling pass run on the GPU box (under gpurun), MODEL env = config (default lenet5, the bench
# workload). Writes small CSV summaries to gpurun_out/ (full .ncu-rep files are exported then
# removed: gpurun copies <= 64 MiB back).
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
M=${MODEL:-lenet5}
N=$(MODEL=$M python tools/profile_step.py --count 2>/dev/null | tail -1)
echo "model $M kernels per eager inference: $N" > gpurun_out/profile_info_$M.txt
# 1) launch list of one inference (cold-cache, serialised: compare shares)
MODEL=$M ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${M}_launches.csv \
    -s "$N" -c "$N" python tools/profile_step.py > /dev/null 2>&1
# 2) full sets of every launch of the dominant kernel classes in the same (second) inference
for k in "AdderRound:40" "ChainStep:40" "chain_kernel:8" "ring_gemm_tc2:8" "ring_gemv:8" "ring_gemm_simt:8"; do
  name=${k%%:*}; cnt=${k##*:}
  MODEL=$M timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
      -k "regex:${name}" -s 0 -c "$cnt" -o "gpurun_out/prof_${M}_${name}" python tools/profile_step.py > /dev/null 2>&1
  if [ -f "gpurun_out/prof_${M}_${name}.ncu-rep" ]; then
    ncu -i "gpurun_out/prof_${M}_${name}.ncu-rep" --page raw --csv > "gpurun_out/prof_${M}_${name}_raw.csv" 2>/dev/null
    rm -f "gpurun_out/prof_${M}_${name}.ncu-rep"
  fi
done
ls -la gpurun_out >> gpurun_out/profile_info_$M.txt
