mkdir -p gpurun_out
NG=$(nvidia-smi -L | wc -l)
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_peer_emu.py -x -q -p no:cacheprovider > gpurun_out/g13_pytest.log 2>&1; echo pytest_rc=$? >> gpurun_out/g13_pytest.log; tail -2 gpurun_out/g13_pytest.log
timeout 1200 python -m pytest tests/test_gpu_multigpu.py -x -q -p no:cacheprovider > gpurun_out/g13_multigpu.log 2>&1; echo multigpu_rc=$? >> gpurun_out/g13_multigpu.log; tail -2 gpurun_out/g13_multigpu.log
for N in 4 2; do
  [ $N -gt $NG ] && continue
  for v in "" "--p2p-pull-all" "--p2p-push"; do
    timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2971$N bench.py --gpus $N --steps 30 --warmup 5 --no-e2e --no-cpu-baseline --exposed-model none $v > gpurun_out/g13_step_n$N.log 2>&1
    echo "== step N=$N $v"; python tools/summ_bench.py < gpurun_out/g13_step_n$N.log 2>/dev/null | head -3
  done
  for rep in 1 2; do
    timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2972$N bench.py --gpus $N --steps 10 --warmup 5 --no-e2e --no-cpu-baseline --workload bert_large --dtype bf16 --exposed-model bert_large > gpurun_out/g13_bf16_n${N}_$rep.log 2>&1
    echo "== bf16 BERT N=$N rep $rep"; python tools/summ_bench.py < gpurun_out/g13_bf16_n${N}_$rep.log 2>/dev/null | grep exposed | cut -c1-140
  done
done
