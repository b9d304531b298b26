# tc3 bring-up: parity tests of both tcgen05 kernels, then kernel timing at ResNet-18 shapes
set -o pipefail
timeout 600 python -m pytest tests/test_gpu_tc_gemm.py -x -q 2>&1 | tail -15 > gpurun_out/tc3_pytest.txt
timeout 600 python tools/tc3_bench.py > gpurun_out/tc3_bench.jsonl 2> gpurun_out/tc3_bench.err
cat gpurun_out/tc3_pytest.txt; cat gpurun_out/tc3_bench.jsonl; tail -3 gpurun_out/tc3_bench.err
