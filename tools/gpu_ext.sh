#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_extensions.py -x -q > gpurun_out/pytest_ext.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_ext.log
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python tools/run_model.py resnet18 --check --iters 2 --no-graph > gpurun_out/cfg_resnet18.log 2>&1; echo "rc=$?" >> gpurun_out/cfg_resnet18.log
timeout 900 python tools/run_model.py bert_base --check --iters 2 --no-graph > gpurun_out/cfg_bert_base.log 2>&1; echo "rc=$?" >> gpurun_out/cfg_bert_base.log
timeout 900 python tools/run_model.py bert_base --weights public --mode pipelined --iters 2 --no-graph > gpurun_out/cfg_bert_base_public.log 2>&1; echo "rc=$?" >> gpurun_out/cfg_bert_base_public.log
