# 4 GPUs: config 4 (bucket-cap sweep vs exposed time) with the final defaults, BERT-large fp32 8x512.
mkdir -p gpurun_out
T4="timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29511"
echo "ARGS: cap-sweep bert N4" > gpurun_out/n4c38_sweep.jsonl
$T4 bench.py --gpus 4 --mode cap-sweep --exposed-model bert_large --exposed-iters 5 --caps 1,5,25,100 >> gpurun_out/n4c38_sweep.jsonl 2>gpurun_out/n4c38.err
