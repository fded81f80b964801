cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python tools/quick_time.py 17669 > gpurun_out/qt17669.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:"k1_|k3_|k4_" -s 6 -c 3 -o gpurun_out/mem17669 python tools/quick_time.py 17669 > gpurun_out/ncu_mem17669.log 2>&1
echo done
