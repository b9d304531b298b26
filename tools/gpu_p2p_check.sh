cd /root/repo; mkdir -p gpurun_out
timeout 1200 python -m pytest -q -m gpu tests -x > gpurun_out/t2.log 2>&1; echo rc=$? >> gpurun_out/t2.log
for i in $(seq 1 15); do
  timeout 300 python -m pytest -x -q -s tests/test_gpu_loopback.py > gpurun_out/flake_$i.log 2>&1
  rc=$?; echo "run $i rc=$rc" >> gpurun_out/flake_summary.log
  [ $rc -eq 0 ] && rm -f gpurun_out/flake_$i.log
done
