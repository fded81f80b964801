cd "$GRAFT_REPO_ROOT"; python tools/kernel_times_full.py 1024 4096 8192 16384 32768 65536 > gpurun_out/ktf.log 2>&1
