mkdir -p gpurun_out
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29514 tools/p2p_trace.py > gpurun_out/g5_trace.log 2>&1
grep '^{' gpurun_out/g5_trace.log
tail -3 gpurun_out/g5_trace.log
