mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_multigpu.py -x -q -p no:cacheprovider > gpurun_out/pytest_multi.log 2>&1; echo pytest=$? >> gpurun_out/pytest_multi.log
rm -f gpurun_out/bench_r11.log
T="timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511"
for args in "--comm-ctas 16" "--comm-ctas 32" "--comm-ctas 64 --timeline-detail" "--comm-ctas 128" "--algo 1 --timeline-detail" "--algo 3 --comm-ctas 32"; do
  echo "ARGS: N2 bert $args" >> gpurun_out/bench_r11.log
  $T bench.py --gpus 2 --steps 10 --warmup 3 --no-e2e --workload bert_large --exposed-model bert_large $args >> gpurun_out/bench_r11.log 2>gpurun_out/bench_r11.err
done
