# Toom depth A/B below 512 words: ring sizes x batches and the d-sweep (F2X_TOOM forces the level count)
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out; rm -f gpurun_out/toomgrid.log
for v in "" "F2X_TOOM=1" "F2X_TOOM=2"; do
  echo "== ${v:-default}" >> gpurun_out/toomgrid.log
  env $v timeout 600 python tools/kernel_times.py 17669:256 17669:512 17669:1024 17669:2048 8000:4096 10000:4096 12323:4096 14000:4096 20000:4096 24000:4096 28000:4096 32000:4096 2>&1 | grep -v -i warn | cut -c1-200 >> gpurun_out/toomgrid.log
  env $v timeout 600 python tools/kernel_times_full.py 4096 8192 16384 2>&1 | grep -v -i warn | cut -c1-200 >> gpurun_out/toomgrid.log
done
cat gpurun_out/toomgrid.log
