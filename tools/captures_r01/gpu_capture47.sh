# 4 GPUs: gradient-as-bucket-view with the copy-engine two-shot in place (CE2, W>2), then one W=4 line.
mkdir -p gpurun_out
timeout 150 python -m pytest tests/test_gpu_grad_view.py -x -q -p no:cacheprovider > gpurun_out/c47_pytest.log 2>&1; echo pytest=$? >> gpurun_out/c47_pytest.log
timeout 75 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29511 \
  bench.py --gpus 4 --grad-view --exposed-model resnet50 --exposed-iters 6 --no-e2e --no-cpu-baseline --steps 100 > gpurun_out/c47_n4_view.json 2> gpurun_out/c47.err
