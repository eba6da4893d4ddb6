mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$? >> gpurun_out/pytest_gpu.log
rm -f gpurun_out/bench_r6.log
B="python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline"
$B > gpurun_out/plain_r6.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:oneshot -s 10 -c 5 -o gpurun_out/prof_w1 $B > gpurun_out/ncu_w1.log 2>&1
T="timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511"
for args in "--algo 2 --comm-ctas 64" "--algo 2 --comm-ctas 128" "--algo 2 --comm-ctas 148" "--algo 3 --comm-ctas 64" "--algo 3 --comm-ctas 128" "--algo 3 --comm-ctas 148" "--algo 2 --comm-ctas 128 --stage-kib 512" "--workload bert_large --algo 2 --comm-ctas 128" "--workload bert_large --algo 3 --comm-ctas 128"; do
  echo "ARGS: N2 $args" >> gpurun_out/bench_r6.log
  $T bench.py --gpus 2 --steps 20 --warmup 5 --no-e2e $args >> gpurun_out/bench_r6.log 2>gpurun_out/bench_r6.err
done
