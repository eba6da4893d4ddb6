mkdir -p gpurun_out
for rep in 1 2; do
  for v in "" "--lanes 2" "--lanes 1" "--comm-ctas 24"; do
    timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29961 bench.py --gpus 4 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --workload bert_large --dtype bf16 --exposed-model bert_large $v > gpurun_out/g20.log 2>&1
    echo "== rep $rep [$v]"; grep '^{' gpurun_out/g20.log | python -c "
import json,sys
d=json.loads(sys.stdin.read()); e=d['exposed']; t=e['timeline_rank0']; p=e['exposed_paired_pct_of_bwd']
print(f\"exposed {e['exposed_pct_of_bwd']:.2f}% paired {p['p10']:.2f}/{p['p50']:.2f}/{p['p90']:.2f} bwd {e['t_bwd_ms']:.2f} tail {t['tail_ms']:.3f} queue {t['max_queue_delay_ms']:.3f} busy {t['comm_busy_ms']:.2f}\")"
    cp gpurun_out/g20.log "gpurun_out/g20_${rep}_$(echo $v | tr -d ' -').log"
  done
done
