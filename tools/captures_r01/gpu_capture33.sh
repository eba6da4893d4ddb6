# 2 GPUs: CE reduce / gather grid (pack-ctas) at W=2.
mkdir -p gpurun_out
T="timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511"
R=gpurun_out/n2c33_bench.jsonl; rm -f $R
for g in 592 1184 2368; do for w in resnet50 bert_large; do
  args="--pack-ctas $g --workload $w --exposed-model none"
  echo "ARGS: N2 $args" >> $R
  $T bench.py --gpus 2 --warmup 5 --no-e2e $args >> $R 2>>gpurun_out/n2c33_bench.err
done; done
