mkdir -p gpurun_out
timeout 1800 python -m pytest tests -x -q -m gpu -p no:cacheprovider > gpurun_out/g14_pytest.log 2>&1; echo pytest_rc=$? >> gpurun_out/g14_pytest.log; tail -3 gpurun_out/g14_pytest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/g14_smoke.log 2>&1; echo smoke_rc=$?; tail -1 gpurun_out/g14_smoke.log
timeout 600 python bench.py > gpurun_out/g14_bench_n1.log 2>&1; echo bench_rc=$?; python tools/summ_bench.py < gpurun_out/g14_bench_n1.log
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/g14_ref_n1.log 2>&1; echo ref_rc=$?; tail -c 600 gpurun_out/g14_ref_n1.log
