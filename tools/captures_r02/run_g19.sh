mkdir -p gpurun_out
timeout 600 python bench.py --steps 50 --warmup 5 --exposed-model none --no-cpu-baseline > gpurun_out/g19_n1.log 2>&1; echo "n1 rc=$?"
grep '^{' gpurun_out/g19_n1.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['e2e'])"
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29951 bench.py --gpus 2 --steps 20 --warmup 5 --exposed-model none > gpurun_out/g19_n2.log 2>&1; echo "n2 rc=$?"
grep '^{' gpurun_out/g19_n2.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['e2e'], d['busbw']['per_algo']['grad_view'])"
