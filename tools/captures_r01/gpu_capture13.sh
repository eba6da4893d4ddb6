# 1 GPU: N=1 contract line + ncu launch list + ncu --set full of the world-1 kernel (current config).
mkdir -p gpurun_out
timeout 600 python bench.py > gpurun_out/c13_n1.json 2> gpurun_out/c13_n1.err
B="python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --exposed-model none"
$B > gpurun_out/c13_plain.log 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c13_launches.csv $B > gpurun_out/c13_ncu_launches.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:local_kernel -s 8 -c 2 -o gpurun_out/c13_prof_local $B > gpurun_out/c13_ncu_full.log 2>&1
$B --workload bert_large > gpurun_out/c13_plain_bert.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:local_kernel -s 8 -c 2 -o gpurun_out/c13_prof_local_bert $B --workload bert_large > gpurun_out/c13_ncu_full_bert.log 2>&1
