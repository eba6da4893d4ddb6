mkdir -p gpurun_out
NG=$(nvidia-smi -L | wc -l)
timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/g16_pytest.log 2>&1; echo pytest_rc=$? >> gpurun_out/g16_pytest.log; tail -2 gpurun_out/g16_pytest.log
for N in 4 2; do
  [ $N -gt $NG ] && continue
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2991$N bench.py --gpus $N --steps 30 --warmup 5 > gpurun_out/g16_bench_n$N.log 2>&1
  echo "== bench N=$N rc=$?"; python tools/summ_bench.py < gpurun_out/g16_bench_n$N.log 2>/dev/null
done
