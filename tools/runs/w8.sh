# experiment: Toom-3 point x = X^32 instead of X^16 (variant build w32): parity + per-kernel times
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out; rm -f gpurun_out/w32.log
cp paper_2201_10473_b200/_build/libf2x.so /tmp/libf2x_default.so
SIZES="57637:16384 17669 35851 28000 20000 24000 12323:4096"

timeout 600 python tools/kernel_times.py $SIZES 2>&1 | grep "^n=" | cut -c1-330 >> gpurun_out/w32.log
timeout 600 python tools/kernel_times_full.py 32768 65536 2>&1 | grep "^d=" | cut -c1-330 >> gpurun_out/w32.log
cp paper_2201_10473_b200/_build_exp/w32/libf2x.so paper_2201_10473_b200/_build/libf2x.so
echo "== w32" >> gpurun_out/w32.log
timeout 600 python tools/kernel_times.py $SIZES 2>&1 | grep "^n=" | cut -c1-330 >> gpurun_out/w32.log
timeout 600 python tools/kernel_times_full.py 32768 65536 2>&1 | grep "^d=" | cut -c1-330 >> gpurun_out/w32.log
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_baseline_batches.py -q 2>&1 | tail -n 6 >> gpurun_out/w32.log
cp /tmp/libf2x_default.so paper_2201_10473_b200/_build/libf2x.so
