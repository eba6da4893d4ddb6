# 2 GPUs: bf16 configs at W=2 with the final code (BERT-large bf16 with exposed time; ResNet-50 bf16).
mkdir -p gpurun_out
T="timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511"
R=gpurun_out/n2c40_bench.jsonl; rm -f $R
for args in "--workload bert_large --dtype bf16 --exposed-model bert_large" "--dtype bf16 --exposed-model resnet50"; do
  echo "ARGS: N2 $args" >> $R
  $T bench.py --gpus 2 --warmup 5 --no-e2e $args >> $R 2>>gpurun_out/n2c40_bench.err
done
