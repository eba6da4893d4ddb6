mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/g24_pytest.log 2>&1; echo pytest_rc=$? >> gpurun_out/g24_pytest.log; tail -3 gpurun_out/g24_pytest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/g24_smoke.log 2>&1; echo smoke_rc=$?
for N in 4 2; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2910$N bench.py --gpus $N --steps 30 --warmup 5 > gpurun_out/g24_bench_n$N.log 2>&1
  echo "== bench N=$N rc=$?"; python tools/summ_bench.py < gpurun_out/g24_bench_n$N.log 2>/dev/null
done
