mkdir -p gpurun_out
NG=$(nvidia-smi -L | wc -l)
# N=1: the driver's bench line, then its ncu launch list and one --set full capture of the top kernel
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/g11_bench_n1.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/g11_launches_n1.csv python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline --exposed-model none > gpurun_out/g11_ncu_list.log 2>&1
echo "n1 rc=$?"; python tools/summ_bench.py < gpurun_out/g11_bench_n1.log | head -3
timeout 900 ncu --set full --clock-control none --import-source on -k regex:local_kernel -s 10 -c 2 -o gpurun_out/g11_local python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline --exposed-model none > gpurun_out/g11_ncu_full.log 2>&1
echo "ncu full rc=$?"
for N in 4 2; do
  [ $N -gt $NG ] && continue
  for W in "--workload bert_large --dtype bf16 --exposed-model bert_large" "--dtype bf16 --exposed-model resnet50"; do
    timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2956$N bench.py --gpus $N --steps 20 --warmup 5 --no-e2e --no-cpu-baseline $W > gpurun_out/g11_bf16_n$N.log 2>&1
    echo "== N=$N $W"; python tools/summ_bench.py < gpurun_out/g11_bf16_n$N.log | grep -v clocks; cp gpurun_out/g11_bf16_n$N.log "gpurun_out/g11_bf16_n${N}_$(echo $W | tr -d ' -' | cut -c1-20).log"
  done
done
N=$([ $NG -ge 4 ] && echo 4 || echo 2)
timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29571 bench.py --gpus $N --mode nosync --workload bert_large --exposed-model bert_large --exposed-iters 20 > gpurun_out/g11_nosync.log 2>&1
echo "nosync rc=$?"; grep '^{' gpurun_out/g11_nosync.log | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print(json.dumps(d.get('nosync')))"
for A in default Ring NVLS; do
  if [ $A = default ]; then unset NCCL_ALGO; else export NCCL_ALGO=$A; fi
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29581 bench.py --gpus $N --mode allreduce-sweep > gpurun_out/g11_sweep_$A.log 2>&1
  echo "sweep $A rc=$?"
done
unset NCCL_ALGO
