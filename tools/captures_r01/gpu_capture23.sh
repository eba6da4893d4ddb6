# 4 GPUs: DDP overlap policy (CE2 for all buckets but the last) vs throughput policy; NVLS at W=4 now.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_multigpu.py -x -q -p no:cacheprovider > gpurun_out/n4c23_pytest.log 2>&1; echo pytest=$? >> gpurun_out/n4c23_pytest.log
T4="timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29511"
R=gpurun_out/n4c23_bench.jsonl; rm -f $R
for args in "--workload bert_large --exposed-model bert_large" "" "--algo 5 --workload bert_large --exposed-model none"; do
  echo "ARGS: N4 $args" >> $R
  $T4 bench.py --gpus 4 --warmup 5 --no-e2e $args >> $R 2>>gpurun_out/n4c23_bench.err
done
