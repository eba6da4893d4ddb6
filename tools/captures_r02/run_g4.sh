mkdir -p gpurun_out
nvidia-smi nvlink -gt d > gpurun_out/g4_nvsmi.log 2>&1; nvidia-smi nvlink -s >> gpurun_out/g4_nvsmi.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_peer_emu.py -x -q -p no:cacheprovider > gpurun_out/g4_pytest.log 2>&1; echo pytest_rc=$? >> gpurun_out/g4_pytest.log
tail -3 gpurun_out/g4_pytest.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29513 tools/p2p_sweep.py > gpurun_out/g4_sweep.log 2>&1
grep '^{' gpurun_out/g4_sweep.log | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print(f\"{d['set']:32s} whole {d['whole_ms']*1e3:7.1f} us {d['whole_busbw']:6.0f} GB/s   kernel {d['kernel_ms']*1e3:7.1f} us {d['kernel_busbw'] or 0:6.0f}\")
"
tail -3 gpurun_out/g4_sweep.log
