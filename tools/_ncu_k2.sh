# ncu full capture of the node kernel at n=17669 (development aid)
python tools/quick_time.py 17669 > gpurun_out/qt.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:k2_node -s 4 -c 1 -o gpurun_out/k2_17669 python tools/quick_time.py 17669 > gpurun_out/ncu_k2.log 2>&1
echo ncu_rc=$?
