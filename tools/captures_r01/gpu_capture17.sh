# 2 GPUs: CE with direct copies issued before the gather wait; threshold 4/16/inf MiB.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_multigpu.py tests/test_gpu_unused.py -x -q -p no:cacheprovider > gpurun_out/n2c17_pytest.log 2>&1; echo pytest=$? >> gpurun_out/n2c17_pytest.log
T="timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511"
R=gpurun_out/n2c17_bench.jsonl; rm -f $R
for args in "--exposed-model none" "--workload bert_large --exposed-model bert_large" "--workload bert_large --exposed-model bert_large --ce-direct-mib 4" "--workload bert_large --exposed-model bert_large --ce-direct-mib 100000" "--ce-direct-mib 4 --exposed-model none"; do
  echo "ARGS: N2 $args" >> $R
  $T bench.py --gpus 2 --warmup 5 --no-e2e $args >> $R 2>>gpurun_out/n2c17_bench.err
done
