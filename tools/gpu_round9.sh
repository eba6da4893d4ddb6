mkdir -p gpurun_out
rm -f gpurun_out/bench_r9.log
for args in "" "--workload bert_large --exposed-model bert_large" "--dtype bf16 --exposed-model none"; do
  echo "ARGS: N1 $args" >> gpurun_out/bench_r9.log
  timeout 400 python bench.py --steps 30 --warmup 5 $args >> gpurun_out/bench_r9.log 2>gpurun_out/bench_r9_n1.err
done
T="timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511"
for args in "--algo 2 --comm-ctas 32" "--algo 2 --comm-ctas 64" "--algo 2 --comm-ctas 128" "--algo 1" "--workload bert_large --exposed-model bert_large --algo 2 --comm-ctas 64" "--workload bert_large --exposed-model bert_large --algo 1"; do
  echo "ARGS: N2 $args" >> gpurun_out/bench_r9.log
  $T bench.py --gpus 2 --steps 20 --warmup 5 --no-e2e $args >> gpurun_out/bench_r9.log 2>gpurun_out/bench_r9.err
done
