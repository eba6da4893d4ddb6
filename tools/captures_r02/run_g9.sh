mkdir -p gpurun_out
NG=$(nvidia-smi -L | wc -l)
echo "gpus=$NG"
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/g9_pytest.log 2>&1; echo pytest_rc=$? >> gpurun_out/g9_pytest.log
tail -3 gpurun_out/g9_pytest.log
for N in 4 2; do
  [ $N -gt $NG ] && continue
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2953$N bench.py --gpus $N --steps 20 --warmup 5 > gpurun_out/g9_bench_n$N.log 2>&1
  echo "== bench N=$N rc=$?"; python tools/summ_bench.py < gpurun_out/g9_bench_n$N.log
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2954$N bench.py --gpus $N --steps 20 --warmup 5 --workload bert_large --exposed-model bert_large --no-e2e > gpurun_out/g9_bert_n$N.log 2>&1
  echo "== bench BERT N=$N rc=$?"; python tools/summ_bench.py < gpurun_out/g9_bert_n$N.log
done
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/g9_bench_n1.log 2>&1; echo "== bench N=1 rc=$?"; python tools/summ_bench.py < gpurun_out/g9_bench_n1.log
