# round-2 first check: GPU tests, ResNet-18 bench pair-evaluated and per-slot
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/r2_first_pytest.txt
timeout 600 python bench.py --model resnet18 --steps 10 --warmup 3 --no-cpu > gpurun_out/r2_first_bench_resnet.json 2> gpurun_out/r2_first_bench_resnet.err
MPCG_PAIR_EVAL=0 MPCG_EPS_FUSE=0 timeout 600 python bench.py --model resnet18 --steps 10 --warmup 3 --no-cpu --no-blocking > gpurun_out/r2_first_bench_resnet_perslot.json 2>&1
tail -3 gpurun_out/r2_first_pytest.txt; cut -c1-600 gpurun_out/r2_first_bench_resnet.json; cut -c1-300 gpurun_out/r2_first_bench_resnet_perslot.json
