#!/bin/bash
# Profiling pass run on the GPU box (under gpurun). Writes only small CSV/JSON summaries to
# gpurun_out/ (full .ncu-rep files are exported to CSV then removed: gpurun copies <= 64 MiB).
set -u
mkdir -p gpurun_out
cd "$(dirname "$0")/.."
N=$(python tools/profile_step.py --count 2>/dev/null | tail -1)
echo "kernels per eager inference: $N" > gpurun_out/profile_info.txt
# 1) launch list of one inference (cold-cache, serialised: compare shares)
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/step_launches.csv \
    -s "$N" -c "$N" python tools/profile_step.py > /dev/null 2>&1
# 2) full sets of the dominant kernel classes in the same inference
for k in "AdderRound:6" "chain_kernel:2" "ring_gemm:4" "MulCombine:3"; do
  name=${k%%:*}; cnt=${k##*:}
  timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
      -k "regex:${name}" -s 0 -c "$cnt" -o "gpurun_out/prof_${name}" python tools/profile_step.py > /dev/null 2>&1
  if [ -f "gpurun_out/prof_${name}.ncu-rep" ]; then
    ncu -i "gpurun_out/prof_${name}.ncu-rep" --page raw --csv > "gpurun_out/prof_${name}_raw.csv" 2>/dev/null
    ncu -i "gpurun_out/prof_${name}.ncu-rep" --page details --csv > "gpurun_out/prof_${name}_details.csv" 2>/dev/null
    rm -f "gpurun_out/prof_${name}.ncu-rep"
  fi
done
ls -la gpurun_out >> gpurun_out/profile_info.txt
