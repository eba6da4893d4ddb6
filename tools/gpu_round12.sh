mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_multigpu.py -x -q -p no:cacheprovider > gpurun_out/pytest_multi.log 2>&1; echo pytest=$? >> gpurun_out/pytest_multi.log
rm -f gpurun_out/bench_r12.log
T="timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511"
for args in "--algo 4" "--workload bert_large --exposed-model bert_large --algo 4 --timeline-detail" "--workload bert_large --exposed-model bert_large --algo 4 --pack-ctas 148" "--workload bert_large --exposed-model bert_large --algo 3 --comm-ctas 16"; do
  echo "ARGS: N2 $args" >> gpurun_out/bench_r12.log
  $T bench.py --gpus 2 --steps 10 --warmup 3 --no-e2e $args >> gpurun_out/bench_r12.log 2>gpurun_out/bench_r12.err
done
