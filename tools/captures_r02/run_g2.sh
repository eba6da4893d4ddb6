mkdir -p gpurun_out
nvidia-smi -L
timeout 1800 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/g2_pytest.log 2>&1; echo pytest_rc=$? >> gpurun_out/g2_pytest.log
tail -5 gpurun_out/g2_pytest.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 20 --warmup 5 > gpurun_out/g2_bench.log 2>&1; echo bench_rc=$?
tail -c 6000 gpurun_out/g2_bench.log
