cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "toom_levels_forced or cyclic_configs or large_full or golden" > gpurun_out/t8.log 2>&1; echo rc=$? >> gpurun_out/t8.log
timeout 900 python -m pytest tests/test_gpu_baseline_batches.py -q -x -k "57637 or 35851 or very_large" >> gpurun_out/t8.log 2>&1; echo rc=$? >> gpurun_out/t8.log
timeout 900 python tools/ab_env.py "F2X_TOOM_WO=0" "F2X_TOOM_WO=512" "F2X_TOOM_WO=1024" "F2X_TOOM_WO=2048" -- 57637:16384 35851 > gpurun_out/ab8.log 2>&1
