# 4 GPUs: host cost of issuing a step (CE2 vs two-shot at W=4); W=2 CE with low-priority streams.
mkdir -p gpurun_out
T4="timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29511"
T2="timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512"
R=gpurun_out/n4c20_bench.jsonl; rm -f $R
for args in "--workload bert_large --exposed-model none" "--algo 7 --workload bert_large --exposed-model none" "--algo 7 --exposed-model none"; do
  echo "ARGS: N4 $args" >> $R
  $T4 bench.py --gpus 4 --warmup 5 --no-e2e $args >> $R 2>>gpurun_out/n4c20_bench.err
done
for args in "--workload bert_large --exposed-model bert_large --low-priority" "--workload bert_large --exposed-model bert_large"; do
  echo "ARGS: N2 $args" >> $R
  CUDA_VISIBLE_DEVICES=0,1 $T2 bench.py --gpus 2 --warmup 5 --no-e2e $args >> $R 2>>gpurun_out/n4c20_bench.err
done
