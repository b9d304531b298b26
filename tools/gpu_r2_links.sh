# round-2: new transport / report / chunking / triple-queue tests, link latency
set -u
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_loopback.py tests/test_gpu_multiprocess.py tests/test_gpu_report.py \
   tests/test_gpu_triple_queue.py tests/test_gpu_parity.py tests/test_gpu_scale.py -m gpu -q 2>&1 | tail -40 > gpurun_out/r2l_pytest.txt
timeout 600 python tools/link_latency.py > gpurun_out/r2l_link_latency.json 2> gpurun_out/r2l_link_latency.err
tail -12 gpurun_out/r2l_pytest.txt; head -c 1500 gpurun_out/r2l_link_latency.json; tail -3 gpurun_out/r2l_link_latency.err
