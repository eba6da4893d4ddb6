# ncu --set full of the copy-engine reduce kernel (peer emulation, W=2, 25 MiB bucket)
mkdir -p gpurun_out
timeout 150 python tools/emu_ce_ncu.py --world 2 > gpurun_out/g31_plain.log 2>&1; rc=$?; echo plain_rc=$rc; tail -1 gpurun_out/g31_plain.log
if [ $rc -eq 0 ]; then
  timeout 240 ncu --set full --clock-control none --import-source on -k regex:ce_reduce --launch-skip 2 -c 1 -f -o gpurun_out/g31_ce_reduce python tools/emu_ce_ncu.py --world 2 > gpurun_out/g31_ncu.log 2>&1; echo ncu_rc=$?; tail -3 gpurun_out/g31_ncu.log
fi
