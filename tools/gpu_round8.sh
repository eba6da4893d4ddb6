mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$? >> gpurun_out/pytest_gpu.log
rm -f gpurun_out/bench_r8.log
for args in "" "--dtype bf16" "--workload bert_large" "--workload bert_large --dtype bf16" "--pack-ctas 148" "--pack-ctas 592" "--pack-ctas 1184"; do
  echo "ARGS: N1 $args" >> gpurun_out/bench_r8.log
  timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e $args >> gpurun_out/bench_r8.log 2>&1
done
B="python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline"
$B > gpurun_out/plain_r8.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:local -s 4 -c 1 -o gpurun_out/prof_local8 $B > gpurun_out/ncu_local8.log 2>&1
