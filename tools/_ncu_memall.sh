# ncu (--set full) of the HBM-side kernels: n=17669 (slice/interp/unslice) and
# n=57637 (Toom evaluation/interpolation, k3, slice/unslice) -- development aid
python tools/quick_time.py 17669 57637 > gpurun_out/qt.log 2>&1 || exit 1
ncu --set full --clock-control none -k regex:"k1_slice|k3_interp|k4_unslice" -s 6 -c 3 -o gpurun_out/mem17669 python tools/quick_time.py 17669 > gpurun_out/ncu_m1.log 2>&1
ncu --set full --clock-control none -k regex:"toom_|k3_interp|k1_slice|k4_unslice" -s 30 -c 10 -o gpurun_out/mem57637 python tools/quick_time.py 57637 > gpurun_out/ncu_m2.log 2>&1
echo done
