# 4 GPUs: throughput policy with 4 lanes x 37 CTAs (the whole GPU) vs 32.
mkdir -p gpurun_out
T4="timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29511"
R=gpurun_out/n4c29_bench.jsonl; rm -f $R
for args in "--comm-ctas 37 --exposed-model none" "--comm-ctas 37 --workload bert_large --exposed-model bert_large" "--comm-ctas 32 --workload bert_large --exposed-model none" "--comm-ctas 37 --workload bert_large --dtype bf16 --exposed-model none"; do
  echo "ARGS: N4 $args" >> $R
  $T4 bench.py --gpus 4 --warmup 5 --no-e2e $args >> $R 2>>gpurun_out/n4c29_bench.err
done
