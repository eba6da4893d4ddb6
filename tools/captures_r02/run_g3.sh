mkdir -p gpurun_out
python tools/nvml_nvlink_probe.py > gpurun_out/g3_nvml.log 2>&1
timeout 900 python -m pytest tests/test_gpu_peer_emu.py tests/test_gpu_parity.py -x -q -p no:cacheprovider > gpurun_out/g3_pytest.log 2>&1; echo pytest_rc=$? >> gpurun_out/g3_pytest.log
tail -3 gpurun_out/g3_pytest.log
B="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 2 --steps 20 --warmup 5 --exposed-model none --no-e2e --no-cpu-baseline"
for v in "" "--p2p-push" "--stage-kib 64" "--stage-kib 32" "--stage-kib 16"; do
  echo "== $v" >> gpurun_out/g3_bench.log
  timeout 300 $B $v 2>&1 | grep '^{' >> gpurun_out/g3_bench.log
done
python - <<'PY'
import json
for line in open("gpurun_out/g3_bench.log"):
    if line.startswith("=="):
        print(line.strip()); continue
    d = json.loads(line)
    print("step_ms", round(d["value"], 4), {k: (v["algo"], round(v["busbw_gbs"]), round(v.get("nonlast", {}).get("busbw_gbs", 0))) for k, v in d["busbw"]["per_algo"].items()})
PY
