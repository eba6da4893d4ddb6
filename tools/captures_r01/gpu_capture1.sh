# Round-1 capture on ONE GPU: GPU tests, smoke, bench (both arms), ncu launch list, ncu full of the top kernel.
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvsmi.txt 2>&1
timeout 900 python -m pytest tests -m "gpu and not multigpu" -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$? >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$? >> gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench_n1.json 2> gpurun_out/bench_n1.err; echo bench=$? >> gpurun_out/bench_n1.err
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 600 python bench.py --workload bert_large --exposed-model bert_large --no-cpu-baseline > gpurun_out/bench_n1_bert.json 2> gpurun_out/bench_n1_bert.err
B="python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --exposed-model none"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $B > gpurun_out/ncu_launches.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:local_kernel -s 8 -c 2 -o gpurun_out/prof_local $B > gpurun_out/ncu_full.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:local_kernel -s 8 -c 2 -o gpurun_out/prof_local_bert $B --workload bert_large > gpurun_out/ncu_full_bert.log 2>&1
ls -la gpurun_out >> gpurun_out/ls.txt
