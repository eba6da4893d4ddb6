# 1 GPU: ncu --set full of pack_kernel / unpack_kernel on a working set larger than L2
# (NCCL path at world 1, BERT-large fp32, 200 MiB cap), the north_star's pack/unpack HBM evidence.
mkdir -p gpurun_out
B="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --exposed-model none --algo 1 --cap-mib 200 --workload bert_large"
$B > gpurun_out/c39_plain.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:"pack_kernel|unpack_kernel" -s 10 -c 4 -o gpurun_out/c39_packunpack $B > gpurun_out/c39_ncu.log 2>&1
