cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_checked_build.py -q -x > gpurun_out/k34_tests.log 2>&1; echo "rc=$?" >> gpurun_out/k34_tests.log
timeout 900 python tools/kernel_times_full.py 4096 8192 16384 > gpurun_out/k34_ab.log 2>&1
