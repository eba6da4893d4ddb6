# N=2: parity (multi-GPU incl. PUSH, front end), PUSH bench variants.
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_multigpu.py tests/test_gpu_unused.py tests/test_gpu_frontend.py -x -q -p no:cacheprovider > gpurun_out/n2c5_pytest.log 2>&1; echo pytest=$? >> gpurun_out/n2c5_pytest.log
T="timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511"
R=gpurun_out/n2c5_bench.jsonl; rm -f $R
for args in "--algo 6" "--algo 6 --comm-ctas 32 --exposed-model none" "--algo 6 --comm-ctas 128 --exposed-model none" "--workload bert_large --exposed-model bert_large --algo 6" "--workload bert_large --exposed-model bert_large --algo 6 --comm-ctas 32" "--workload bert_large --exposed-model bert_large --algo 2"; do
  echo "ARGS: $args" >> $R
  $T bench.py --gpus 2 --warmup 5 $args >> $R 2>>gpurun_out/n2c5_bench.err
done
