for L in paper_2209_13643_b200/lib/libmpcg.so paper_2209_13643_b200/lib/libmpcg_seeded.so; do
  echo "== $L $(MPCG_LIB=$L timeout 600 python tools/run_model.py bert_base --mode blocking --iters 3 2>&1 | grep -oE '"graph_ms": [0-9.]+' | head -1) $(MPCG_LIB=$L timeout 600 python tools/run_model.py lenet5 --mode blocking --iters 5 2>&1 | grep -oE '"graph_ms": [0-9.]+' | head -1)"
done
