mkdir -p gpurun_out
NG=$(nvidia-smi -L | wc -l)
for N in 4 2; do
  [ $N -gt $NG ] && continue
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2961$N tools/p2p_trace.py > gpurun_out/g12_trace_n$N.log 2>&1
  echo "== trace N=$N"; grep '^{' gpurun_out/g12_trace_n$N.log | grep '"rank": 0'
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2962$N tools/step_trace.py resnet50 > gpurun_out/g12_step_n$N.log 2>&1
  echo "== step trace N=$N"; grep '^{' gpurun_out/g12_step_n$N.log
  for v in "--overlap-policy 1" "--overlap-policy 2" "--overlap-policy 2 --p2p-push" "--overlap-policy 2 --comm-ctas 16"; do
    timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2963$N bench.py --gpus $N --steps 10 --warmup 5 --no-e2e --no-cpu-baseline --workload bert_large --dtype bf16 --exposed-model bert_large $v > gpurun_out/g12_bf16_n$N.log 2>&1
    echo "== bf16 BERT N=$N $v"; python tools/summ_bench.py < gpurun_out/g12_bf16_n$N.log 2>/dev/null | grep exposed | cut -c1-160
    cp gpurun_out/g12_bf16_n$N.log "gpurun_out/g12_bf16_n${N}_$(echo $v | tr -d ' -').log"
  done
done
export NCCL_ALGO="allreduce:nvls"
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29591 bench.py --gpus $NG --mode allreduce-sweep > gpurun_out/g12_sweep_NVLS.log 2>&1
echo "sweep NVLS rc=$?"
