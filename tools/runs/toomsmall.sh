# Toom depth at small batches of the large ring sizes (the per-level latency term of the planner)
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out; rm -f gpurun_out/toomsmall.log
SIZES="35851:32 35851:256 35851:1024 57637:32 57637:256 57637:1024 57637:4096 17669:32 24000:256 24000:2048 32000:1024 32000:2048 22000:1024 22000:2048 26000:2048 14000:2048 15000:3072"
for v in "" "F2X_TOOM=0" "F2X_TOOM=1" "F2X_TOOM=2" "F2X_TOOM=3"; do
  echo "== ${v:-default}" >> gpurun_out/toomsmall.log
  env $v timeout 900 python tools/kernel_times.py $SIZES 2>&1 | grep "^n=" | cut -c1-60 >> gpurun_out/toomsmall.log
done
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -n 4 >> gpurun_out/toomsmall.log
