# 1 GPU: world-1 kernel at 4736 vs 9472 CTAs (ResNet-50 / BERT-large), 3 repeats each.
mkdir -p gpurun_out
R=gpurun_out/c28_local.jsonl; rm -f $R
for rep in 1 2 3; do for g in 4736 9472; do for w in resnet50 bert_large; do
  echo "ARGS: pack-ctas $g $w rep $rep" >> $R
  timeout 300 python bench.py --workload $w --pack-ctas $g --exposed-model none --no-cpu-baseline --no-e2e >> $R 2>>gpurun_out/c28.err
done; done; done
