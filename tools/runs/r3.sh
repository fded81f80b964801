cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "toom_levels_forced or cyclic_configs or large_full or golden" > gpurun_out/t3.log 2>&1; echo rc=$? >> gpurun_out/t3.log
timeout 600 python tools/ab_env.py "F2X_TOOM_EVAL=levels" "" -- 57637:16384 35851 > gpurun_out/ab3.log 2>&1
