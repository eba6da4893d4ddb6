# 4 GPUs: communication stream priority (high = default vs lowest) for the exposed time of a real backward.
mkdir -p gpurun_out
T4="timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29511"
R=gpurun_out/n4c19_bench.jsonl; rm -f $R
for args in "--workload bert_large --exposed-model bert_large" "--workload bert_large --exposed-model bert_large --low-priority" "--algo 7 --workload bert_large --exposed-model bert_large --low-priority" "--low-priority"; do
  echo "ARGS: N4 $args" >> $R
  $T4 bench.py --gpus 4 --warmup 5 --no-e2e $args >> $R 2>>gpurun_out/n4c19_bench.err
done
