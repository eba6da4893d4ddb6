mkdir -p gpurun_out
NG=$(nvidia-smi -L | wc -l)
echo "gpus=$NG"
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "pull or resnet or toy" > gpurun_out/g8_parity.log 2>&1; echo parity_rc=$? >> gpurun_out/g8_parity.log; tail -2 gpurun_out/g8_parity.log
timeout 1200 python -m pytest tests/test_gpu_multigpu.py -x -q -p no:cacheprovider > gpurun_out/g8_multigpu.log 2>&1; echo multigpu_rc=$? >> gpurun_out/g8_multigpu.log; tail -2 gpurun_out/g8_multigpu.log
for N in 4 2; do
  [ $N -gt $NG ] && continue
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2952$N tools/p2p_sweep.py --sets quick > gpurun_out/g8_sweep_n$N.log 2>&1
  echo "== sweep N=$N"; grep '^{' gpurun_out/g8_sweep_n$N.log | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print(f\"{d['set']:16s} whole {d['whole_ms']*1e3:7.1f} us {d['whole_busbw']:6.0f} GB/s   kernel {d['kernel_ms']*1e3:7.1f} us {d['kernel_busbw'] or 0:6.0f}\")
"
  for v in "" "--comm-ctas 37" "--p2p-push" "--lanes 2 --comm-ctas 74"; do
    timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2953$N bench.py --gpus $N --steps 20 --warmup 5 --exposed-model none --no-e2e $v > gpurun_out/g8_bench_n$N.log 2>&1
    echo "== bench N=$N $v"; python tools/summ_bench.py < gpurun_out/g8_bench_n$N.log | head -3
  done
done
