# N=2: parity (multi-GPU incl. NVLS + find_unused), CE multi-stream copies, NVLS bench, sweep.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_multigpu.py tests/test_gpu_unused.py -x -q -p no:cacheprovider > gpurun_out/n2c4_pytest.log 2>&1; echo pytest=$? >> gpurun_out/n2c4_pytest.log
T="timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511"
R=gpurun_out/n2c4_bench.jsonl; rm -f $R
for args in "--algo 4 --ce-streams 1 --exposed-model none" "--algo 4 --ce-streams 4" "--algo 4 --ce-streams 8 --exposed-model none" "--algo 5" "--workload bert_large --exposed-model bert_large --algo 4" "--workload bert_large --exposed-model bert_large --algo 5" "--workload bert_large --exposed-model none --algo 4 --ce-streams 8"; do
  echo "ARGS: $args" >> $R
  $T bench.py --gpus 2 --warmup 5 $args >> $R 2>>gpurun_out/n2c4_bench.err
done
$T bench.py --gpus 2 --mode allreduce-sweep > gpurun_out/n2c4_sweep.jsonl 2>>gpurun_out/n2c4_bench.err
