# 4 GPUs: two-shot pipeline stages, pack/unpack HBM efficiency at a 200 MiB cap (NCCL path), config 5 at N=4, smoke.
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/c15_smoke.log 2>&1; echo smoke=$? >> gpurun_out/c15_smoke.log
T4="timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29511"
R=gpurun_out/n4c15_bench.jsonl; rm -f $R
for args in "--stage-kib 256" "--stage-kib 1024" "--workload bert_large --stage-kib 1024" "--algo 1 --cap-mib 200 --workload bert_large" "--algo 1 --cap-mib 200"; do
  echo "ARGS: N4 $args" >> $R
  $T4 bench.py --gpus 4 --warmup 5 --no-e2e --exposed-model none $args >> $R 2>>gpurun_out/n4c15_bench.err
done
echo "ARGS: nosync bert N4" > gpurun_out/n4c15_nosync.jsonl
$T4 bench.py --gpus 4 --mode nosync --exposed-model bert_large --exposed-iters 6 >> gpurun_out/n4c15_nosync.jsonl 2>>gpurun_out/n4c15_bench.err
