# 1 GPU: local-kernel U / grid experiment (N=1 contract workload, ResNet-50 and BERT)
mkdir -p gpurun_out
R=gpurun_out/c9_local.jsonl; rm -f $R
for u in 8 4; do for g in 1184 2368 4736; do for w in resnet50 bert_large; do
  echo "ARGS: U=$u pack-ctas $g $w" >> $R
  B200DDP_LOCAL_U=$u timeout 300 python bench.py --workload $w --pack-ctas $g --exposed-model none --no-cpu-baseline --no-e2e >> $R 2>>gpurun_out/c9.err
done; done; done
