# GPU tests + per-kernel times (ring sizes and the d-sweep) -> gpurun_out/
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x -rfEs > gpurun_out/gputest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gputest.log
timeout 300 python tools/kernel_times.py 17669 35851 57637:16384 12323:256 > gpurun_out/ktimes.log 2>&1
timeout 600 python tools/kernel_times_full.py 1024 4096 16384 65536 >> gpurun_out/ktimes.log 2>&1
