cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 1500 python tools/ab_env.py "F2X_TOOM=0" "F2X_TOOM=1" "F2X_TOOM=2" "F2X_TOOM=3" -- 17669 35851 > gpurun_out/toomlev.log 2>&1
for v in 0 1 2; do echo "== F2X_TOOM=$v" >> gpurun_out/toomlev.log; F2X_TOOM=$v python tools/kernel_times_full.py 16384 32768 2>/dev/null | grep "^d=" >> gpurun_out/toomlev.log; done
