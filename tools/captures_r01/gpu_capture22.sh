# 2 GPUs: one-shot (4 lanes x 32 CTAs, last bucket on 148) vs the CE default at W=2.
mkdir -p gpurun_out
T="timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511"
R=gpurun_out/n2c22_bench.jsonl; rm -f $R
for args in "--algo 2" "--algo 2 --workload bert_large --exposed-model bert_large" "--algo 3 --exposed-model none" ""; do
  echo "ARGS: N2 $args" >> $R
  $T bench.py --gpus 2 --warmup 5 --no-e2e $args >> $R 2>>gpurun_out/n2c22_bench.err
done
