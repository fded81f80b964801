cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x -k "toom or cyclic_configs or large_full or golden" > gpurun_out/t12.log 2>&1; echo rc=$? >> gpurun_out/t12.log
timeout 600 python tools/kernel_times.py 35851 57637:16384 > gpurun_out/kt12.log 2>&1
