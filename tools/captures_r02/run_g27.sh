mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_peer_emu.py -x -q -p no:cacheprovider > gpurun_out/g27_pytest.log 2>&1; echo pytest_rc=$?; tail -1 gpurun_out/g27_pytest.log
for rep in 1 2; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 2982$rep bench.py --gpus 2 --steps 20 --warmup 5 --no-e2e --no-cpu-baseline --exposed-model none > gpurun_out/g27_n2.log 2>&1
echo "== N=2 rep $rep rc=$?"; python tools/summ_bench.py < gpurun_out/g27_n2.log 2>/dev/null | head -3
done
