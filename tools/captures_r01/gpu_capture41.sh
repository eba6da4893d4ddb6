# 2 GPUs: BERT-large bf16 exposed time at W=2: CE (default) with a smaller kernel grid, one-shot, two-shot.
mkdir -p gpurun_out
T="timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511"
R=gpurun_out/n2c41_bench.jsonl; rm -f $R
for args in "--pack-ctas 296" "--algo 2" "--algo 3"; do
  echo "ARGS: N2 bf16 $args" >> $R
  $T bench.py --gpus 2 --warmup 5 --no-e2e --workload bert_large --dtype bf16 --exposed-model bert_large $args >> $R 2>>gpurun_out/n2c41_bench.err
done
