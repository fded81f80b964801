cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
: > gpurun_out/toomlev2.log
for v in 2 3; do echo "== F2X_TOOM=$v" >> gpurun_out/toomlev2.log; F2X_TOOM=$v python tools/kernel_times_full.py 65536 2>/dev/null | grep "^d=" >> gpurun_out/toomlev2.log; done
timeout 900 python tools/ab_env.py "F2X_TOOM=2" "F2X_TOOM=3" -- 57637:16384 >> gpurun_out/toomlev2.log 2>&1
python tools/kernel_times_full.py 32768 2>/dev/null | grep "^d=" >> gpurun_out/toomlev2.log
