mkdir -p gpurun_out
NG=$(nvidia-smi -L | wc -l)
timeout 900 python -m pytest tests/test_gpu_peer_emu.py tests/test_gpu_parity.py tests/test_gpu_grad_view.py -x -q -p no:cacheprovider > gpurun_out/g18_pytest.log 2>&1; echo pytest_rc=$? >> gpurun_out/g18_pytest.log; tail -2 gpurun_out/g18_pytest.log
timeout 1500 python -m pytest tests/test_gpu_multigpu.py -x -q -p no:cacheprovider > gpurun_out/g18_multigpu.log 2>&1; echo multigpu_rc=$? >> gpurun_out/g18_multigpu.log; tail -2 gpurun_out/g18_multigpu.log
for N in 4 2; do
  [ $N -gt $NG ] && continue
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2993$N bench.py --gpus $N --steps 20 --warmup 5 --no-e2e --no-cpu-baseline --exposed-model none > gpurun_out/g18_bench_n$N.log 2>&1
  echo "== bench N=$N rc=$?"; python tools/summ_bench.py < gpurun_out/g18_bench_n$N.log 2>/dev/null | head -3
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2994$N bench.py --gpus $N --steps 20 --warmup 5 --no-e2e --no-cpu-baseline --grad-view > gpurun_out/g18_view_n$N.log 2>&1
  echo "== grad-view bench N=$N rc=$?"; python tools/summ_bench.py < gpurun_out/g18_view_n$N.log 2>/dev/null | grep -v clocks
done
