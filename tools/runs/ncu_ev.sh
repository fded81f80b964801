cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python tools/quick_time.py 57637 > gpurun_out/qt_ev.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:"toom_eval|k1_slice|k4_uns" -s 7 -c 3 -o gpurun_out/ev57637 python tools/quick_time.py 57637 > gpurun_out/ncu_ev.log 2>&1
echo done
