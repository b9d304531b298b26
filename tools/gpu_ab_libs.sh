# A/B of library builds (MPCG_LIB): ReLU (8.4M) adder time, LeNet-5 / ResNet-18 / BERT-base graph latency
for L in ${LIBS:-lib_ab/libmpcg_mb4.so lib_ab/libmpcg_mb5.so}; do
  echo "== $L"
  MPCG_LIB=$L timeout 300 python tools/relu_probe.py --time
  echo "lenet $(MPCG_LIB=$L timeout 300 python tools/run_model.py lenet5 --mode pipelined --iters 5 2>&1 | grep -oE '"graph_ms": [0-9.]+' | head -1) r18 $(MPCG_LIB=$L timeout 300 python tools/run_model.py resnet18 --mode pipelined --iters 3 2>&1 | grep -oE '"graph_ms": [0-9.]+' | head -1) bert $(MPCG_LIB=$L timeout 600 python tools/run_model.py bert_base --mode pipelined --iters 3 2>&1 | grep -oE '"graph_ms": [0-9.]+' | head -1)"
done
