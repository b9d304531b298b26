# bench A/B of the current build (ResNet-18 default workload) + pool-mode parity tests
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_triple_queue.py tests/test_gpu_parity.py -m gpu -q 2>&1 | tail -4 > gpurun_out/r2ab_pytest.txt
for i in 1 2; do
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu --no-variants --no-blocking > gpurun_out/r2ab_bench_$i.json 2> gpurun_out/r2ab_bench_$i.err
done
cat gpurun_out/r2ab_pytest.txt
python - <<'P'
import json
for i in (1,2):
    d=json.load(open(f"gpurun_out/r2ab_bench_{i}.json"))
    print(round(d["ms_per_step"],3), [(r["kernel"], round(r["device_ms_per_step"],2), round(r["frac"],3)) for r in d["rooflines"]], d["clocks"])
P
