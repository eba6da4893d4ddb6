# 2 GPUs: full GPU test suite, N=1 and N=2 default bench lines, then configs 4/5 sweeps at N=2.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/c8_pytest.log 2>&1; echo pytest=$? >> gpurun_out/c8_pytest.log
timeout 600 python bench.py > gpurun_out/c8_n1.json 2> gpurun_out/c8_n1.err
timeout 600 python bench.py --workload bert_large --exposed-model bert_large --no-cpu-baseline > gpurun_out/c8_n1_bert.json 2>> gpurun_out/c8_n1.err
T="timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511"
$T bench.py --gpus 2 > gpurun_out/c8_n2.json 2> gpurun_out/c8_n2.err
$T bench.py --gpus 2 --workload bert_large --exposed-model bert_large > gpurun_out/c8_n2_bert.json 2>> gpurun_out/c8_n2.err
$T bench.py --gpus 2 --workload bert_large --exposed-model bert_large --wire-bf16 > gpurun_out/c8_n2_bert_wire.json 2>> gpurun_out/c8_n2.err
$T bench.py --gpus 2 --impl reference > gpurun_out/c8_n2_ref.json 2>> gpurun_out/c8_n2.err
bash tools/gpu_capture6.sh
