# A/B of library builds (MPCG_LIB): ReLU (8.4M) adder time and BERT-base / LeNet-5 latency
for L in ${LIBS:-lib_ab/libmpcg_old.so paper_2209_13643_b200/lib/libmpcg.so}; do
  echo "== $L"
  MPCG_LIB=$L timeout 300 python tools/relu_probe.py --time
  MPCG_LIB=$L timeout 600 python tools/run_model.py bert_base --mode blocking --iters 3 2>&1 | grep -oE '"graph_ms": [0-9.]+' | head -1
  MPCG_LIB=$L timeout 300 python tools/run_model.py lenet5 --mode blocking --iters 5 2>&1 | grep -oE '"graph_ms": [0-9.]+' | head -1
  MPCG_LIB=$L timeout 300 python tools/run_model.py resnet18 --mode blocking --iters 3 2>&1 | grep -oE '"graph_ms": [0-9.]+' | head -1
done
