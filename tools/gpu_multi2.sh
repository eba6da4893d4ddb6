mkdir -p gpurun_out
nvidia-smi topo -m > gpurun_out/topo.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_multigpu.py -x -q -p no:cacheprovider > gpurun_out/pytest_multi.log 2>&1; echo pytest=$? >> gpurun_out/pytest_multi.log
T="timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511"
for args in "" "--algo 1" "--comm-ctas 8" "--comm-ctas 16" "--comm-ctas 64" "--comm-ctas 128" "--dtype bf16" "--workload bert_large" "--workload bert_large --algo 1" "--workload bert_large --dtype bf16"; do
  echo "ARGS: $args" >> gpurun_out/bench_n2.log
  $T bench.py --gpus 2 --steps 20 --warmup 5 --no-e2e $args >> gpurun_out/bench_n2.log 2>gpurun_out/bench_n2.err
done
