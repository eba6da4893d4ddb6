# Configs 4 and 5 (BASELINE.json): bucket-cap sweep vs exposed time, and no_sync every 1/2/4/8, at N=2.
mkdir -p gpurun_out
T="timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511"
R=gpurun_out/n2c6_sweeps.jsonl; rm -f $R
for args in "--exposed-model resnet50" "--exposed-model resnet50 --exposed-batch 16" "--exposed-model bert_large" "--exposed-model bert_large --exposed-seq 128"; do
  echo "ARGS: cap-sweep $args" >> $R
  $T bench.py --gpus 2 --mode cap-sweep --exposed-iters 6 $ALGO $args >> $R 2>>gpurun_out/n2c6.err
done
echo "ARGS: nosync bert" >> $R
$T bench.py --gpus 2 --mode nosync --exposed-model bert_large --exposed-iters 6 $ALGO >> $R 2>>gpurun_out/n2c6.err
