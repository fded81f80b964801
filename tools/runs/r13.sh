cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 900 python tools/ab_env.py "" "F2X_TOOM_SEQ=100" "F2X_TOOM_SEQ=1000" -- 35851 > gpurun_out/ab13.log 2>&1
