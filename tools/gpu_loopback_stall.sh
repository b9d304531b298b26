#!/bin/bash
# Reproduce the rare eager-loopback stall: the bench's one-party loopback variant
# at ResNet-18 scale, several times, with the link's post trace and a Python stack dump.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for i in $(seq 1 ${N:-4}); do
  MPCG_LINK_DEBUG=1 timeout 300 python -c "
import faulthandler, sys, runpy
faulthandler.dump_traceback_later(240, exit=True)
sys.argv = ['bench.py', '--one-party-variants', '--no-cpu', '--no-blocking', '--steps', '4', '--warmup', '3']
runpy.run_path('bench.py', run_name='__main__')
" > gpurun_out/stall_$i.out 2> gpurun_out/stall_$i.err
  echo "run $i rc=$?" >> gpurun_out/stall_summary.log
done
