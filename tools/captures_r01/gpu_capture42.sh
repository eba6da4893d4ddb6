# 2 GPUs: final suite after the bf16 overlap policy; BERT-large bf16 / fp32 exposed with the front end's defaults.
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/c42_pytest.log 2>&1; echo pytest=$? >> gpurun_out/c42_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/c42_smoke.log 2>&1; echo smoke=$? >> gpurun_out/c42_smoke.log
T="timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511"
R=gpurun_out/n2c42_bench.jsonl; rm -f $R
for args in "--workload bert_large --dtype bf16 --exposed-model bert_large" "--workload bert_large --exposed-model bert_large"; do
  echo "ARGS: N2 $args" >> $R
  $T bench.py --gpus 2 --warmup 5 --no-e2e $args >> $R 2>>gpurun_out/n2c42_bench.err
done
