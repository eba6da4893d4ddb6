# 4 GPUs: BERT-large bf16 exposed time, overlap policy (default in DDP) vs throughput policy.
mkdir -p gpurun_out
T4="timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29511"
R=gpurun_out/n4c34_bench.jsonl; rm -f $R
for args in "--throughput-policy" ""; do
  echo "ARGS: N4 bf16 $args" >> $R
  $T4 bench.py --gpus 4 --warmup 5 --no-e2e --workload bert_large --dtype bf16 --exposed-model bert_large --timeline-detail $args >> $R 2>>gpurun_out/n4c34_bench.err
done
