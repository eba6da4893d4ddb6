# host watchdog added: new test first, then the driver's 1-GPU commands
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/g29_build.log 2>&1; echo build_rc=$?
timeout 120 python -m pytest tests/test_gpu_peer_emu.py -x -q -p no:cacheprovider -k watchdog 2>&1 | tail -3
timeout 1500 python -m pytest tests -x -q -m gpu -p no:cacheprovider > gpurun_out/g29_pytest.log 2>&1; echo pytest_rc=$?; tail -2 gpurun_out/g29_pytest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/g29_smoke.log 2>&1; echo smoke_rc=$?; tail -1 gpurun_out/g29_smoke.log
timeout 600 python bench.py > gpurun_out/g29_bench.log 2>&1; echo bench_rc=$?; python tools/summ_bench.py < gpurun_out/g29_bench.log
