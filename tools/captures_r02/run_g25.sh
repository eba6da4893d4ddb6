mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/g25_build.log 2>&1; echo build_rc=$?
timeout 1800 python -m pytest tests -x -q -m gpu -p no:cacheprovider > gpurun_out/g25_pytest.log 2>&1; echo pytest_rc=$?; tail -2 gpurun_out/g25_pytest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/g25_smoke.log 2>&1; echo smoke_rc=$?; tail -1 gpurun_out/g25_smoke.log
timeout 900 python bench.py > gpurun_out/g25_bench.log 2>&1; echo bench_rc=$?; python tools/summ_bench.py < gpurun_out/g25_bench.log
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/g25_ref.log 2>&1; echo ref_rc=$?; grep '^{' gpurun_out/g25_ref.log | cut -c1-200
