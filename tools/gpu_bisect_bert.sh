for L in ${LIBS:-lib_ab/libmpcg_head.so lib_ab/libmpcg_ni.so}; do
  echo "== $L bert $(MPCG_LIB=$L timeout 600 python tools/run_model.py bert_base --mode blocking --iters 3 2>&1 | grep -oE '"graph_ms": [0-9.]+' | head -1) lenet $(MPCG_LIB=$L timeout 600 python tools/run_model.py lenet5 --mode blocking --iters 5 2>&1 | grep -oE '"graph_ms": [0-9.]+' | head -1) r18 $(MPCG_LIB=$L timeout 600 python tools/run_model.py resnet18 --mode blocking --iters 3 2>&1 | grep -oE '"graph_ms": [0-9.]+' | head -1)"
done
