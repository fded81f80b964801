cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 900 python tools/ab_env.py "F2X_TOOM=2 F2X_TOOM_LEAF=16" "F2X_TOOM=2 F2X_TOOM_LEAF=24" -- 35851 > gpurun_out/leaf35851.log 2>&1
timeout 900 python tools/ab_env.py "F2X_TOOM=3 F2X_TOOM_LEAF=18" "F2X_TOOM=3 F2X_TOOM_LEAF=24" -- 57637:16384 > gpurun_out/leaf57637.log 2>&1
