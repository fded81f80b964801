cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python tools/quick_time.py 17669 > gpurun_out/qt17669.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:"k1_|k3_|k4_|k2_" -s 4 -c 4 -o gpurun_out/all17669 python tools/quick_time.py 17669 > gpurun_out/ncu_all17669.log 2>&1
echo done
