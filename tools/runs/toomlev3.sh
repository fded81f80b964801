# Toom depth A/B after the round-2 interpolation changes (F2X_TOOM forces the level count)
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
for v in "" "F2X_TOOM=3" "F2X_TOOM=2" "F2X_TOOM=1"; do
  echo "== ${v:-default}" >> gpurun_out/toomlev3.log
  env $v timeout 900 python tools/kernel_times_full.py 32768 65536 >> gpurun_out/toomlev3.log 2>&1
  env $v timeout 600 python tools/kernel_times.py 35851 57637:16384 >> gpurun_out/toomlev3.log 2>&1
done
