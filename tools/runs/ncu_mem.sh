# ncu --set full captures of the memory-side kernels at n=57637 x 16384 and
# n=35851 x 4096, plus n=35851's launch list and node-kernel capture
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python tools/quick_time.py 57637 35851 > gpurun_out/qt.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:"toom|k1_|k3_|k4_" -s 7 -c 6 -o gpurun_out/mem57637 python tools/quick_time.py 57637 > gpurun_out/ncu_mem57637.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launch_list_35851.csv python tools/quick_time.py 35851 > gpurun_out/ncu_ll35851.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"toom|k1_|k3_|k4_|k2_" -s 9 -c 9 -o gpurun_out/all35851 python tools/quick_time.py 35851 > gpurun_out/ncu_all35851.log 2>&1
echo done
