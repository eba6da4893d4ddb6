mkdir -p gpurun_out
nvidia-smi topo -m > gpurun_out/topo4.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_multigpu.py -x -q -p no:cacheprovider > gpurun_out/pytest_multi4.log 2>&1; echo pytest=$? >> gpurun_out/pytest_multi4.log
rm -f gpurun_out/bench_r10.log
T="timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29511"
for args in "" "--algo 2" "--algo 3 --comm-ctas 128" "--algo 1" "--workload bert_large --exposed-model bert_large" "--workload bert_large --exposed-model bert_large --algo 1" "--workload bert_large --exposed-model none --algo 3 --comm-ctas 128"; do
  echo "ARGS: N4 $args" >> gpurun_out/bench_r10.log
  $T bench.py --gpus 4 --steps 20 --warmup 5 --no-e2e $args >> gpurun_out/bench_r10.log 2>gpurun_out/bench_r10.err
done
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29512 tools/nccl_ref.py > gpurun_out/nccl_ref4.txt 2>&1
