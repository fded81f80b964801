# ncu captures of the memory-side kernels at n=17669 (development aid)
python tools/quick_time.py 17669 > gpurun_out/qt.log 2>&1 || exit 1
ncu --set full --clock-control none -k regex:"k1_slice|k3_interp|k4_unslice" -s 6 -c 3 -o gpurun_out/mem17669 python tools/quick_time.py 17669 > gpurun_out/ncu_mem.log 2>&1
echo ncu_rc=$?
