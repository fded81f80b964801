# --set full capture of every kernel of one n=35851 x 4096 call (profiles/r2/all35851.*)
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python tools/quick_time.py 35851 > gpurun_out/qt35851.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:"toom|k1_|k3_|k4_|k2_" -s 7 -c 7 -o gpurun_out/all35851 python tools/quick_time.py 35851 > gpurun_out/ncu_all35851.log 2>&1
echo done
