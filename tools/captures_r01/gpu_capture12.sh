# 4 GPUs: CE2 parity (world 2 and 4) + CE2 bench at N=4 and N=2.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_multigpu.py tests/test_gpu_unused.py -x -q -p no:cacheprovider > gpurun_out/n4c12_pytest.log 2>&1; echo pytest=$? >> gpurun_out/n4c12_pytest.log
T4="timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29511"
T2="timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512"
R=gpurun_out/n4c12_bench.jsonl; rm -f $R
for args in "" "--workload bert_large --exposed-model bert_large" "--algo 7" "--algo 7 --workload bert_large --exposed-model bert_large" "--workload bert_large --dtype bf16 --exposed-model none"; do
  echo "ARGS: N4 $args" >> $R
  $T4 bench.py --gpus 4 --warmup 5 --no-e2e $args >> $R 2>>gpurun_out/n4c12_bench.err
done
for args in "--algo 7 --workload bert_large --exposed-model bert_large"; do
  echo "ARGS: N2 $args" >> $R
  CUDA_VISIBLE_DEVICES=0,1 $T2 bench.py --gpus 2 --warmup 5 --no-e2e $args >> $R 2>>gpurun_out/n4c12_bench.err
done
