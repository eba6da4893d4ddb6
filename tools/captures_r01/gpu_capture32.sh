# 4 GPUs, final round-1 lines at N=4 (defaults): ResNet-50 and BERT-large, with exposed time.
mkdir -p gpurun_out
T4="timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29511"
$T4 bench.py --gpus 4 > gpurun_out/c32_n4.json 2> gpurun_out/c32_n4.err
$T4 bench.py --gpus 4 --workload bert_large --exposed-model bert_large > gpurun_out/c32_n4_bert.json 2>> gpurun_out/c32_n4.err
$T4 bench.py --gpus 4 --workload bert_large --dtype bf16 --exposed-model bert_large > gpurun_out/c32_n4_bert_bf16.json 2>> gpurun_out/c32_n4.err
