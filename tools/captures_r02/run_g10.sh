mkdir -p gpurun_out
NG=$(nvidia-smi -L | wc -l)
for N in 4 2; do
  [ $N -gt $NG ] && continue
  for rep in 1 2; do
    for v in "" "--last-on-lane"; do
      timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2955$N bench.py --gpus $N --steps 30 --warmup 5 --no-e2e --no-cpu-baseline $v > gpurun_out/g10_n${N}_${rep}${v}.log 2>&1
      echo "== N=$N rep=$rep $v"; python tools/summ_bench.py < gpurun_out/g10_n${N}_${rep}${v}.log | grep -v clocks
    done
  done
done
