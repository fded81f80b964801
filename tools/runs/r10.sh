cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "toom_levels_forced or cyclic_configs or large_full or golden" > gpurun_out/t10.log 2>&1; echo rc=$? >> gpurun_out/t10.log
timeout 900 python -m pytest tests/test_gpu_baseline_batches.py -q -x -k "57637 or 35851 or very_large or dsweep" >> gpurun_out/t10.log 2>&1; echo rc=$? >> gpurun_out/t10.log
timeout 600 python tools/kernel_times.py 57637:16384 35851 > gpurun_out/kt10.log 2>&1
