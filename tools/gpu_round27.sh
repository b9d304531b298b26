#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
MPCG_EPS_FUSE=0 timeout 300 python tools/ab_eps_fuse.py > gpurun_out/ab0.log 2>&1
MPCG_EPS_FUSE=1 timeout 300 python tools/ab_eps_fuse.py > gpurun_out/ab1.log 2>&1
