# ncu captures of the Toom-path memory kernels at n=57637 (development aid)
python tools/quick_time.py 57637 > gpurun_out/qt.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:"toom_interp_seq|toom_eval_level|k3_interp" -s 21 -c 7 -o gpurun_out/toom57637 python tools/quick_time.py 57637 > gpurun_out/ncu_toom.log 2>&1
echo ncu_rc=$?
