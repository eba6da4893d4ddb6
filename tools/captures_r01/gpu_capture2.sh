# Round-1 capture on TWO GPUs: multi-GPU parity, NVLink probe, NCCL reference busBW, bench N=2 per algorithm.
mkdir -p gpurun_out
nvidia-smi topo -m > gpurun_out/n2_topo.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_multigpu.py -x -q -p no:cacheprovider > gpurun_out/n2_pytest.log 2>&1; echo pytest=$? >> gpurun_out/n2_pytest.log
timeout 120 tools/nvlink_probe 256 > gpurun_out/n2_nvlink_probe.txt 2>&1
T="timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511"
NCCL_DEBUG=INFO NCCL_DEBUG_SUBSYS=INIT,TUNING $T tools/nccl_ref.py > gpurun_out/n2_nccl_ref.txt 2>&1
R=gpurun_out/n2_bench.jsonl; rm -f $R
for args in "" "--algo 1 --exposed-model none" "--algo 3 --exposed-model none" "--algo 4" "--workload bert_large --exposed-model bert_large" "--workload bert_large --exposed-model bert_large --algo 1" "--workload bert_large --exposed-model bert_large --algo 4" "--workload bert_large --dtype bf16 --exposed-model none"; do
  echo "ARGS: $args" >> $R
  $T bench.py --gpus 2 --warmup 5 $args >> $R 2>>gpurun_out/n2_bench.err
done
$T bench.py --gpus 2 --impl reference --steps 3 --warmup 1 > gpurun_out/n2_ref.json 2>>gpurun_out/n2_bench.err
