mkdir -p gpurun_out
set -x
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$? >> gpurun_out/pytest_gpu.log
for args in "" "--algo 1" "--pack-ctas 148" "--pack-ctas 592" "--dtype bf16" "--workload bert_large" "--workload bert_large --dtype bf16"; do
  echo "ARGS: $args" >> gpurun_out/bench2.log
  timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline $args >> gpurun_out/bench2.log 2>&1
done
