# bf16 BERT-large W=4 exposed time: default vs gradient_as_bucket_view (fused in-place two-shot everywhere)
mkdir -p gpurun_out/g28
i=0
for cfg in view default view default; do
  i=$((i+1)); extra=""; [ $cfg = view ] && extra="--grad-view"
  timeout 170 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 2998$i bench.py --gpus 4 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --workload bert_large --dtype bf16 --exposed-model bert_large $extra > gpurun_out/g28/out$i.log 2>&1
  echo "run $i $cfg rc=$? t=$SECONDS"; grep '^{' gpurun_out/g28/out$i.log | python -c "
import json,sys
d=json.loads(sys.stdin.read()); e=d['exposed']; p=e['exposed_paired_pct_of_bwd']
print(f\"value {d['value']:.3f} exposed {e['exposed_pct_of_bwd']:.2f}% paired {p['p10']:.2f}/{p['p50']:.2f}/{p['p90']:.2f} bwd {e['t_bwd_ms']:.2f} algos {sorted(set(d.get('algos',[])))}\")" 2>&1 | tail -1
done
