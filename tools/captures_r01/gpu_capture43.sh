# 4 GPUs, final code: default lines (ResNet-50 fp32, BERT-large fp32 and bf16 with exposed time).
mkdir -p gpurun_out
T4="timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29511"
$T4 bench.py --gpus 4 > gpurun_out/c43_n4.json 2> gpurun_out/c43.err
$T4 bench.py --gpus 4 --workload bert_large --exposed-model bert_large --no-e2e > gpurun_out/c43_n4_bert.json 2>> gpurun_out/c43.err
$T4 bench.py --gpus 4 --workload bert_large --dtype bf16 --exposed-model bert_large --no-e2e > gpurun_out/c43_n4_bert_bf16.json 2>> gpurun_out/c43.err
