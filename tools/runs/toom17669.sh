# Toom depth A/B at the headline size with the final round-2 passes (F2X_TOOM forces the level count)
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
for v in "" "F2X_TOOM=1" "F2X_TOOM=2"; do
  echo "== ${v:-default}" >> gpurun_out/toom17669.log
  env $v timeout 600 python tools/kernel_times.py 17669 12323:256 17669:16384 >> gpurun_out/toom17669.log 2>&1
done
cat gpurun_out/toom17669.log
