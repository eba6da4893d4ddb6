# 4 GPUs: multi-GPU parity at world 4, bench N=4 per algorithm, allreduce sweep.
mkdir -p gpurun_out
timeout 300 python bench.py --exposed-model none --no-cpu-baseline > gpurun_out/n4_n1check.json 2>&1
nvidia-smi topo -m > gpurun_out/n4_topo.txt 2>&1
timeout 1200 python -m pytest tests/test_gpu_multigpu.py -x -q -p no:cacheprovider > gpurun_out/n4_pytest.log 2>&1; echo pytest=$? >> gpurun_out/n4_pytest.log
T="timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29511"
NCCL_DEBUG=INFO NCCL_DEBUG_SUBSYS=INIT,TUNING $T tools/nccl_ref.py > gpurun_out/n4_nccl_ref.txt 2>&1
R=gpurun_out/n4_bench.jsonl; rm -f $R
for args in "" "--workload bert_large --exposed-model bert_large" "--algo 3 --exposed-model none" "--algo 3 --workload bert_large --exposed-model bert_large" "--algo 1 --exposed-model none" "--algo 4 --exposed-model none" "--algo 6 --exposed-model none" "--algo 4 --workload bert_large --exposed-model bert_large" "--algo 5 --comm-ctas 128 --exposed-model none"; do
  echo "ARGS: $args" >> $R
  $T bench.py --gpus 4 --warmup 5 $args >> $R 2>>gpurun_out/n4_bench.err
done
$T bench.py --gpus 4 --mode allreduce-sweep > gpurun_out/n4_sweep.jsonl 2>>gpurun_out/n4_bench.err
