mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$? >> gpurun_out/pytest_gpu.log
rm -f gpurun_out/bench_r5.log
T="timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511"
for args in "--algo 2 --comm-ctas 16" "--algo 2 --comm-ctas 32" "--algo 2 --comm-ctas 64" "--algo 2 --comm-ctas 128" "--algo 3 --comm-ctas 32" "--algo 3 --comm-ctas 64" "--algo 3 --comm-ctas 128" "--workload bert_large --algo 2 --comm-ctas 64" "--workload bert_large --algo 3 --comm-ctas 64"; do
  echo "ARGS: N2 $args" >> gpurun_out/bench_r5.log
  $T bench.py --gpus 2 --steps 20 --warmup 5 --no-e2e $args >> gpurun_out/bench_r5.log 2>gpurun_out/bench_r5.err
done
