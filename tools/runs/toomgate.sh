# where the group-count gate of the sub-512-word Toom plans belongs: 64 / 80 / 96 / 112 groups
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out; rm -f gpurun_out/toomgate.log
SIZES="17669:2048 17669:2560 17669:3072 17669:3584 20000:2048 20000:3072 28000:2048 28000:3072 12323:2048 12323:3072 24000:1024 28000:1024 20000:1024"
for v in "F2X_TOOM=0" "F2X_TOOM=1" "F2X_TOOM=2" "F2X_TOOM=3"; do
  echo "== ${v:-default}" >> gpurun_out/toomgate.log
  env $v timeout 900 python tools/kernel_times.py $SIZES 2>&1 | grep "^n=" | cut -c1-60 >> gpurun_out/toomgate.log
done
