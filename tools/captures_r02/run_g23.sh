mkdir -p gpurun_out
for N in 4 2; do
  for v in "--overlap-policy 1" "--overlap-policy 2"; do
    timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2998$N bench.py --gpus $N --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --workload bert_large --exposed-model bert_large $v > gpurun_out/g23.log 2>&1
    echo "== N=$N [$v]"; grep '^{' gpurun_out/g23.log | python -c "
import json,sys
d=json.loads(sys.stdin.read()); e=d['exposed']; t=e['timeline_rank0']; p=e['exposed_paired_pct_of_bwd']
print(f\"exposed {e['exposed_pct_of_bwd']:.2f}% paired {p['p10']:.2f}/{p['p50']:.2f}/{p['p90']:.2f} bwd {e['t_bwd_ms']:.2f} tail {t['tail_ms']:.3f} algos {sorted(set(e['bucket_algos']))}\")"
    cp gpurun_out/g23.log "gpurun_out/g23_n${N}_$(echo $v | tr -d ' -').log"
    timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2999$N bench.py --gpus $N --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --exposed-model resnet50 $v > gpurun_out/g23r.log 2>&1
    echo "== ResNet N=$N [$v]"; grep '^{' gpurun_out/g23r.log | python -c "
import json,sys
d=json.loads(sys.stdin.read()); e=d['exposed']; t=e['timeline_rank0']; p=e['exposed_paired_pct_of_bwd']
print(f\"exposed {e['exposed_pct_of_bwd']:.2f}% paired {p['p10']:.2f}/{p['p50']:.2f}/{p['p90']:.2f} bwd {e['t_bwd_ms']:.2f} tail {t['tail_ms']:.3f}\")"
  done
done
