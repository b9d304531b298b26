cd /root/repo; mkdir -p gpurun_out
timeout 1500 python -m pytest -q -m gpu tests -x > gpurun_out/chk_tests.log 2>&1; echo "rc=$?" >> gpurun_out/chk_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/chk_smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/chk_bench.log 2>&1; echo "rc=$?" >> gpurun_out/chk_bench.log
