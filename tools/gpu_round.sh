#!/bin/bash
# one gpurun call: GPU tests, per-kernel times, a short bench (logs in gpurun_out/)
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -rfEs > gpurun_out/gputest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gputest.log
timeout 300 python tools/kernel_times.py 17669 35851 57637:16384 12323:256 > gpurun_out/ktimes.log 2>&1
timeout 600 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
