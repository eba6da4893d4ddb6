mkdir -p gpurun_out/g21
export PYTHONFAULTHANDLER=1
for rep in 1 2 3; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 2997$rep --log-dir gpurun_out/g21/rep$rep --tee 3 bench.py --gpus 4 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --workload bert_large --dtype bf16 --exposed-model bert_large > gpurun_out/g21/out$rep.log 2>&1
  echo "rep $rep rc=$?"; grep '^{' gpurun_out/g21/out$rep.log | python -c "
import json,sys
d=json.loads(sys.stdin.read()); e=d['exposed']; p=e['exposed_paired_pct_of_bwd']
print(f\"value {d['value']:.3f} exposed {e['exposed_pct_of_bwd']:.2f}% paired {p['p10']:.2f}/{p['p50']:.2f}/{p['p90']:.2f} bwd {e['t_bwd_ms']:.2f}\")" 2>/dev/null
  grep -h -B2 -A25 "Fatal Python error\|Segmentation" gpurun_out/g21/out$rep.log | head -60
done
