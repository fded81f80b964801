cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 900 python tools/split_streams.py 17669:4096 35851:4096 57637:16384 12323:256 --splits 1,2,3,4,6 > gpurun_out/split.log 2>&1
F2X_WS_BUDGET=$((48<<30)) timeout 600 python tools/dsweep.py 16384 32768 65536 > gpurun_out/dsweep_ws48.log 2>&1
timeout 600 python tools/dsweep.py 16384 32768 65536 > gpurun_out/dsweep_ws8.log 2>&1
