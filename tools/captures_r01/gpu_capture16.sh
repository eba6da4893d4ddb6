# 2 GPUs: bidirectional copy-engine probe; CE2 vs CE at W=2 (ResNet-50); default lines.
mkdir -p gpurun_out
timeout 120 tools/nvlink_probe 256 > gpurun_out/n2c16_probe.txt 2>&1
T="timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511"
R=gpurun_out/n2c16_bench.jsonl; rm -f $R
for args in "" "--algo 7" "--workload bert_large --dtype bf16 --exposed-model bert_large"; do
  echo "ARGS: N2 $args" >> $R
  $T bench.py --gpus 2 --warmup 5 $args >> $R 2>>gpurun_out/n2c16_bench.err
done
