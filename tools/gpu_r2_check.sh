# round-2 check: new parity tests, full GPU suite, default bench line (ResNet-18)
set -o pipefail
timeout 900 python -m pytest tests/test_gpu_scale.py tests/test_gpu_parity.py -m gpu -x -q -k "not vgg16_whole" 2>&1 | tail -25 > gpurun_out/r2_check_new.txt
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -25 > gpurun_out/r2_check_all.txt
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/r2_check_bench.json 2> gpurun_out/r2_check_bench.err
tail -5 gpurun_out/r2_check_new.txt; tail -5 gpurun_out/r2_check_all.txt; tail -3 gpurun_out/r2_check_bench.err; cut -c1-400 gpurun_out/r2_check_bench.json
