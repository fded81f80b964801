# parity tests (test_gpu_parity.py) + per-kernel times -> gpurun_out/
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_checked_build.py -q -x > gpurun_out/quick_tests.log 2>&1; echo "rc=$?" >> gpurun_out/quick_tests.log
timeout 300 python tools/kernel_times.py 17669 35851 57637:16384 12323:256 > gpurun_out/ktimes.log 2>&1
timeout 600 python tools/kernel_times_full.py 1024 4096 >> gpurun_out/ktimes.log 2>&1
