# 4 GPUs: lanes (multi-stream P2P/NVLS) vs 1 lane, COMM_CTAS for exposure; parity with lanes.
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_multigpu.py -x -q -p no:cacheprovider > gpurun_out/n4c11_pytest.log 2>&1; echo pytest=$? >> gpurun_out/n4c11_pytest.log
T="timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29511"
R=gpurun_out/n4c11_bench.jsonl; rm -f $R
for args in "--exposed-model none --lanes 1" "--exposed-model none" "--exposed-model none --lanes 4 --comm-ctas 32" "--workload bert_large --exposed-model none --lanes 1" "--workload bert_large --exposed-model bert_large" "--workload bert_large --exposed-model bert_large --comm-ctas 32 --lanes 4" "--workload bert_large --exposed-model bert_large --comm-ctas 16 --lanes 4" "--algo 5 --workload bert_large --exposed-model none" "--algo 5 --exposed-model none"; do
  echo "ARGS: $args" >> $R
  $T bench.py --gpus 4 --warmup 5 --no-e2e $args >> $R 2>>gpurun_out/n4c11_bench.err
done
