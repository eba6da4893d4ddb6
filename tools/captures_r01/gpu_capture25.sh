# 2 GPUs: 4 vectors per source for 2-source reductions (CE reduce at W=2): parity + bench.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_multigpu.py tests/test_gpu_parity.py -x -q -p no:cacheprovider > gpurun_out/n2c25_pytest.log 2>&1; echo pytest=$? >> gpurun_out/n2c25_pytest.log
T="timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511"
R=gpurun_out/n2c25_bench.jsonl; rm -f $R
for args in "" "--workload bert_large --exposed-model bert_large"; do
  echo "ARGS: N2 $args" >> $R
  $T bench.py --gpus 2 --warmup 5 --no-e2e $args >> $R 2>>gpurun_out/n2c25_bench.err
done
