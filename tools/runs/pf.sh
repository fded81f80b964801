cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 1500 python tools/ab_env.py "F2X_PREFETCH_AHEAD=0" "F2X_PREFETCH_AHEAD=296" "F2X_PREFETCH_AHEAD=444" "F2X_PREFETCH_AHEAD=888" -- 17669 35851 57637:16384 > gpurun_out/pf.log 2>&1
