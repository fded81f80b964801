# resident-root Toom interpolation: parity + A/B against the separate k3_interp<1> pass
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_baseline_batches.py -q -x -k "configs_vs_oracle or toom_levels_forced or full_size_properties or large_full or exact_baseline or golden" > gpurun_out/kroot_tests.log 2>&1; echo "rc=$?" >> gpurun_out/kroot_tests.log
timeout 600 python tools/ab_env.py "" "F2X_KROOT=0" -- 57637:16384 57637:2048 > gpurun_out/kroot_ab.log 2>&1
