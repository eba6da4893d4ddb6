mkdir -p gpurun_out
NG=$(nvidia-smi -L | wc -l)
N=$([ $NG -ge 4 ] && echo 4 || echo 2)
timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29601 bench.py --gpus $N --mode cap-sweep --exposed-model bert_large --exposed-iters 30 > gpurun_out/g17_cap_bert.log 2>&1
echo "cap bert rc=$?"
timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29602 bench.py --gpus $N --mode cap-sweep --exposed-model bert_large --exposed-seq 128 --exposed-iters 30 > gpurun_out/g17_cap_bert128.log 2>&1
echo "cap bert128 rc=$?"
timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29603 bench.py --gpus $N --mode cap-sweep --exposed-model resnet50 --exposed-batch 16 --exposed-iters 30 > gpurun_out/g17_cap_resnet16.log 2>&1
echo "cap resnet16 rc=$?"
for f in gpurun_out/g17_cap_*.log; do echo "== $f"; grep '^{' $f | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); p=d['exposed_paired_pct_of_bwd']
    print(f\"cap {d['bucket_cap_mib']:>6} MiB buckets {d['buckets']:3d} bwd {d['t_bwd_ms']:6.2f} ms exposed {d['exposed_ms']:6.3f} ms = {d['exposed_pct_of_bwd']:5.2f}% (paired {p['p10']:.2f}/{p['p50']:.2f}/{p['p90']:.2f}) no-overlap {d.get('exposed_no_overlap_ms', 0):.3f} ms\")
"; done
