# --set full captures of the slicing / unslicing passes at d=1024 (configs[4], 4M products)
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python tools/kernel_times_full.py 1024 > gpurun_out/ktf1024.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:"k1_|k4_" -s 2 -c 2 -o gpurun_out/mem1024 python tools/kernel_times_full.py 1024 > gpurun_out/ncu_mem1024.log 2>&1
echo done
