for p in 0 1; do
  echo "pdl=$p lenet $(MPCG_PDL=$p timeout 300 python tools/run_model.py lenet5 --mode pipelined --iters 5 2>&1 | grep -oE '"graph_ms": [0-9.]+' | head -1) mlp $(MPCG_PDL=$p timeout 300 python tools/run_model.py mlp --mode pipelined --iters 5 2>&1 | grep -oE '"graph_ms": [0-9.]+' | head -1) r18 $(MPCG_PDL=$p timeout 300 python tools/run_model.py resnet18 --mode pipelined --iters 3 2>&1 | grep -oE '"graph_ms": [0-9.]+' | head -1)"
done
