# after templating the fused evaluation on the innermost point: parity + per-kernel times
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_baseline_batches.py tests/test_checked_build.py -q 2>&1 | tail -n 4 > gpurun_out/evalwl.log
timeout 600 python tools/kernel_times.py 57637:16384 17669 35851 30000 2>&1 | grep "^n=" | cut -c1-330 >> gpurun_out/evalwl.log
cat gpurun_out/evalwl.log
