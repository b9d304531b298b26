set -o pipefail
MPCG_TC2_TRACE=1 timeout 300 python tools/tc2_trace.py 131072 576 64 > gpurun_out/trace_l1.txt 2>&1
MPCG_TC2_TRACE=1 timeout 300 python tools/tc2_trace.py 8192 1152 128 > gpurun_out/trace_l2.txt 2>&1
MPCG_TC2_TRACE=1 timeout 300 python tools/tc2_trace.py 2048 4608 512 > gpurun_out/trace_l4.txt 2>&1
tail -3 gpurun_out/trace_l1.txt gpurun_out/trace_l2.txt gpurun_out/trace_l4.txt
