# 2 GPUs, final verification after the last changes: full GPU suite, smoke, N=1 / N=2 contract lines.
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/c36_pytest.log 2>&1; echo pytest=$? >> gpurun_out/c36_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/c36_smoke.log 2>&1; echo smoke=$? >> gpurun_out/c36_smoke.log
timeout 600 python bench.py > gpurun_out/c36_n1.json 2> gpurun_out/c36_n1.err
T="timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511"
$T bench.py --gpus 2 > gpurun_out/c36_n2.json 2> gpurun_out/c36_n2.err
