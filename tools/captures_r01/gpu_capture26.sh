# 2 GPUs: full GPU suite after the last-bucket fix; N=1 contract line.
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/c26_pytest.log 2>&1; echo pytest=$? >> gpurun_out/c26_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/c26_smoke.log 2>&1; echo smoke=$? >> gpurun_out/c26_smoke.log
timeout 600 python bench.py > gpurun_out/c26_n1.json 2> gpurun_out/c26_n1.err
