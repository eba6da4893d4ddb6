mkdir -p gpurun_out
python tools/emu_twoshot.py 4 twoshot pull > gpurun_out/g22_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:pull_twoshot -s 2 -c 2 -o gpurun_out/g22_pull python tools/emu_twoshot.py 4 twoshot pull > gpurun_out/g22_ncu.log 2>&1
echo "rc=$?"; tail -3 gpurun_out/g22_ncu.log
