#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 python tools/lenet_knobs.py lenet5 > gpurun_out/knobs_nopdl.log 2>&1
MPCG_PDL=1 timeout 600 python tools/lenet_knobs.py lenet5 > gpurun_out/knobs_pdl.log 2>&1
MPCG_PDL=1 timeout 600 python tools/lenet_knobs.py mlp > gpurun_out/knobs_pdl_mlp.log 2>&1
timeout 600 python tools/lenet_knobs.py mlp > gpurun_out/knobs_nopdl_mlp.log 2>&1
