for L in paper_2209_13643_b200/lib/libmpcg.so lib_ab/libmpcg_cg.so; do
  echo "$L lenet $(MPCG_LIB=$L timeout 300 python tools/run_model.py lenet5 --mode pipelined --iters 5 2>&1 | grep -oE '"graph_ms": [0-9.]+' | head -1) mlp $(MPCG_LIB=$L timeout 300 python tools/run_model.py mlp --mode pipelined --iters 5 2>&1 | grep -oE '"graph_ms": [0-9.]+' | head -1)"
done
