cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x > gpurun_out/t11.log 2>&1; echo rc=$? >> gpurun_out/t11.log
timeout 600 python tools/kernel_times.py 17669 35851 57637:16384 12323:256 > gpurun_out/kt11.log 2>&1
python tools/dsweep.py > gpurun_out/ds11.log 2>&1
