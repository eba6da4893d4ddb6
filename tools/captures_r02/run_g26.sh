mkdir -p gpurun_out
for v in "--ce-streams 3" "--ce-streams 1" "--ce-streams 3"; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29811 bench.py --gpus 4 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --workload bert_large --exposed-model bert_large $v > gpurun_out/g26.log 2>&1
  echo "== [$v]"; grep '^{' gpurun_out/g26.log | python -c "
import json,sys
d=json.loads(sys.stdin.read()); e=d['exposed']; t=e['timeline_rank0']; p=e['exposed_paired_pct_of_bwd']
print(f\"exposed {e['exposed_pct_of_bwd']:.2f}% paired {p['p10']:.2f}/{p['p50']:.2f}/{p['p90']:.2f} bwd {e['t_bwd_ms']:.2f} tail {t['tail_ms']:.3f} queue {t['max_queue_delay_ms']:.3f} ce2 busbw {d['busbw']['per_algo']['ce2']['busbw_gbs']:.0f}\")"
done
