# Dry run of the N>1 path on one GPU: 2 and 4 ranks (1 and 2 pairs), one party per process over
# the socket link, all on cuda:0; plus the reference arm under torchrun
for n in 2 4; do
  MPCG_SAME_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
    --master-port $((29500 + n)) bench.py --gpus $n --steps 3 --warmup 3 --model lenet5 --no-cpu --no-blocking \
    > gpurun_out/multi_dry_$n.json 2> gpurun_out/multi_dry_$n.err
  echo "n=$n rc=$?"; cut -c1-400 gpurun_out/multi_dry_$n.json; grep -iE "error|Traceback" gpurun_out/multi_dry_$n.err | head -5
done
