# innermost Toom level at x = X^8 (F2X_TOOM_WLAST=8) vs X^16: parity and per-kernel times
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out; rm -f gpurun_out/wlast.log
F2X_TOOM_WLAST=8 timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_baseline_batches.py -q 2>&1 | tail -n 6 >> gpurun_out/wlast.log
SIZES="57637:16384 17669 35851 28000 20000 24000 30000 22000 26000 32000 12323:4096 57637:1024"
for v in "" "F2X_TOOM_WLAST=16" "F2X_TOOM_WLAST=8"; do
  echo "== ${v:-default}" >> gpurun_out/wlast.log
  env $v timeout 600 python tools/kernel_times.py $SIZES 2>&1 | grep "^n=" | cut -c1-250 >> gpurun_out/wlast.log
  env $v timeout 600 python tools/kernel_times_full.py 16384 32768 65536 2>&1 | grep "^d=" | cut -c1-250 >> gpurun_out/wlast.log
done
