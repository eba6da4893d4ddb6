# N=2: CE direct-copy threshold sweep (synthetic + exposed), then the local-kernel probe on GPU 0.
mkdir -p gpurun_out
T="timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511"
R=gpurun_out/n2c7_bench.jsonl; rm -f $R
for d in 1 4 16 10000; do
  for w in "" "--workload bert_large"; do
    args="--algo 4 --ce-direct-mib $d $w --exposed-model none"
    echo "ARGS: $args" >> $R
    $T bench.py --gpus 2 --warmup 5 $args >> $R 2>>gpurun_out/n2c7_bench.err
  done
  args="--algo 4 --ce-direct-mib $d --workload bert_large --exposed-model bert_large --no-e2e"
  echo "ARGS: $args" >> $R
  $T bench.py --gpus 2 --warmup 5 $args >> $R 2>>gpurun_out/n2c7_bench.err
done
timeout 300 tools/local_probe > gpurun_out/local_probe.txt 2>&1
timeout 300 tools/local_probe 1340567552 > gpurun_out/local_probe_bert.txt 2>&1
