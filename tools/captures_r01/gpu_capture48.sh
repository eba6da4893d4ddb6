# 2 GPUs: multi-GPU parity at world 2 after the CE2 / view refactor (all algorithms incl. CE2 with copies).
mkdir -p gpurun_out
timeout 140 python -m pytest "tests/test_gpu_multigpu.py::test_multigpu_parity[2]" tests/test_gpu_grad_view.py -x -q -p no:cacheprovider > gpurun_out/c48_pytest.log 2>&1; echo pytest=$? >> gpurun_out/c48_pytest.log
