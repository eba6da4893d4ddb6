mkdir -p gpurun_out
B="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline"
$B > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $B > gpurun_out/ncu_launches.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:oneshot -s 12 -c 3 -o gpurun_out/prof_oneshot $B > gpurun_out/ncu_full.log 2>&1
for args in "" "--algo 1"; do
  echo "ARGS: $args" >> gpurun_out/bench3.log
  timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline $args >> gpurun_out/bench3.log 2>&1
done
