mkdir -p gpurun_out
NG=$(nvidia-smi -L | wc -l)
timeout 900 python -m pytest tests/test_gpu_peer_emu.py tests/test_gpu_parity.py -x -q -p no:cacheprovider > gpurun_out/g15_pytest.log 2>&1; echo pytest_rc=$? >> gpurun_out/g15_pytest.log; tail -2 gpurun_out/g15_pytest.log
timeout 1500 python -m pytest tests -m multigpu -x -q -p no:cacheprovider > gpurun_out/g15_multigpu.log 2>&1; echo multigpu_rc=$? >> gpurun_out/g15_multigpu.log; tail -2 gpurun_out/g15_multigpu.log
for N in 4 2; do
  [ $N -gt $NG ] && continue
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2981$N bench.py --gpus $N --steps 30 --warmup 5 > gpurun_out/g15_bench_n$N.log 2>&1
  echo "== bench N=$N rc=$?"; python tools/summ_bench.py < gpurun_out/g15_bench_n$N.log 2>/dev/null
done
export NCCL_ALGO="allreduce:nvls,ring" NCCL_DEBUG=INFO NCCL_DEBUG_SUBSYS=TUNING
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29591 bench.py --gpus $NG --mode allreduce-sweep > gpurun_out/g15_sweep_NVLS.log 2>&1
echo "sweep NVLS rc=$?"; grep -c "NVLS" gpurun_out/g15_sweep_NVLS.log
