# 2 GPUs, final code of the session: full GPU suite + smoke, N=1 contract line, N=2 default line.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/c46_pytest.log 2>&1; echo pytest=$? >> gpurun_out/c46_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/c46_smoke.log 2>&1; echo smoke=$? >> gpurun_out/c46_smoke.log
timeout 300 python bench.py > gpurun_out/c46_n1.json 2> gpurun_out/c46_n1.err
T2="timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511"
$T2 bench.py --gpus 2 > gpurun_out/c46_n2.json 2> gpurun_out/c46_n2.err
