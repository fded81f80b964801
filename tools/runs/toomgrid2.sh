# planner regret check: default pick vs forced Toom depth over ring sizes (batch 4096 / 16384)
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out; rm -f gpurun_out/toomgrid2.log
SIZES="9000 10000 11000 12323 13000 14000 15000 16000 17669 19000 20000 22000 24000 26000 28000 30000 32000 35851 17669:16384 12323:16384 24000:16384"
for v in "" "F2X_TOOM=0" "F2X_TOOM=1" "F2X_TOOM=2" "F2X_TOOM=3"; do
  echo "== ${v:-default}" >> gpurun_out/toomgrid2.log
  env $v timeout 900 python tools/kernel_times.py $SIZES 2>&1 | grep "^n=" | cut -c1-60 >> gpurun_out/toomgrid2.log
done
python tools/kernel_times_full.py 16384 2>&1 | grep "^d=" | cut -c1-200 >> gpurun_out/toomgrid2.log
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_baseline_batches.py -q -x 2>&1 | tail -n 3 >> gpurun_out/toomgrid2.log
cat gpurun_out/toomgrid2.log
