# 1 GPU: ncu --set full of the P2P kernels in emulation (W ranks in one cooperative launch).
mkdir -p gpurun_out
python tools/emu_twoshot.py 4 twoshot > gpurun_out/c27_plain.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:twoshot -s 2 -c 2 -o gpurun_out/c27_twoshot python tools/emu_twoshot.py 4 twoshot > gpurun_out/c27_ncu.log 2>&1
python tools/emu_twoshot.py 2 oneshot > gpurun_out/c27_plain2.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:oneshot -s 2 -c 2 -o gpurun_out/c27_oneshot python tools/emu_twoshot.py 2 oneshot > gpurun_out/c27_ncu2.log 2>&1
