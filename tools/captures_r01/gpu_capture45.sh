# 2 GPUs: gradient-as-bucket-view with the copy-engine exchange in place (W=2 default) vs copies.
mkdir -p gpurun_out
timeout 400 python -m pytest tests/test_gpu_grad_view.py -x -q > gpurun_out/c45_pytest.log 2>&1
T2="timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511"
for w in resnet50 bert_large; do
  $T2 bench.py --gpus 2 --workload $w --exposed-model $w --no-e2e --no-cpu-baseline > gpurun_out/c45_n2_${w}_ce.json 2>> gpurun_out/c45.err
  $T2 bench.py --gpus 2 --workload $w --grad-view --exposed-model $w --no-e2e --no-cpu-baseline > gpurun_out/c45_n2_${w}_view.json 2>> gpurun_out/c45.err
done
