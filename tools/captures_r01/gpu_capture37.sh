# 4 GPUs: round-robin NCCL communicators (paper Fig. 12, rr1 vs rr3 vs rr5) on BERT-large and ResNet-50.
mkdir -p gpurun_out
T4="timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29511"
R=gpurun_out/n4c37_bench.jsonl; rm -f $R
for k in 1 3 5; do
  for args in "--algo 1 --nccl-comms $k --workload bert_large --exposed-model bert_large" "--algo 1 --nccl-comms $k --exposed-model none"; do
    echo "ARGS: N4 $args" >> $R
    $T4 bench.py --gpus 4 --warmup 5 --no-e2e $args >> $R 2>>gpurun_out/n4c37_bench.err
  done
done
