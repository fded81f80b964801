# ncu capture of the level-3 Toom interpolation at n=57637 (development aid)
python tools/quick_time.py 57637 > gpurun_out/qt.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:"toom_interp_seq" -s 3 -c 1 -o gpurun_out/seq57637 python tools/quick_time.py 57637 > gpurun_out/ncu_seq.log 2>&1
echo ncu_rc=$?
