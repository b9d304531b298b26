# per-kernel launch lists of one BERT-base inference: an older tree (lib_ab/wt_*) vs HEAD
(cd lib_ab/wt_dbad20d && N=$(MODEL=bert_base python tools/profile_step.py --count 2>/dev/null | tail -1) && \
  MODEL=bert_base timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file ../../gpurun_out/bert_old_launches.csv -s "$N" -c "$N" python tools/profile_step.py > /dev/null 2>&1)
MODELS=bert_base bash tools/gpu_launches.sh
ls -la gpurun_out/bert_old_launches.csv gpurun_out/bert_base_launches.csv
