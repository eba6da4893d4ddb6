mkdir -p gpurun_out
./tools/nvlink_probe 256 > gpurun_out/nvlink_probe.txt 2>&1
./tools/nvlink_probe 25 > gpurun_out/nvlink_probe25.txt 2>&1
NCCL_DEBUG=INFO timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 tools/nccl_ref.py > gpurun_out/nccl_ref.txt 2> gpurun_out/nccl_ref.err
