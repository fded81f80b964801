cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python tools/quick_time.py 57637 > gpurun_out/qt_wo.log 2>&1 || exit 1
F2X_TOOM_WO=1024 ncu --set full --clock-control none --import-source on -k regex:"toom_interp" -s 3 -c 3 -o gpurun_out/wo57637 python tools/quick_time.py 57637 > gpurun_out/ncu_wo.log 2>&1
echo done
