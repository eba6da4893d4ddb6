# final code (host watchdog) on 2 GPUs: the whole -m gpu suite incl. the multigpu tests
mkdir -p gpurun_out
timeout 400 python -m pytest tests -x -q -m gpu -p no:cacheprovider > gpurun_out/g30_pytest.log 2>&1; echo pytest_rc=$?; tail -2 gpurun_out/g30_pytest.log
