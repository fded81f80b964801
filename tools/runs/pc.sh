cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python tools/percall_latency.py > gpurun_out/pc.log 2>&1
timeout 900 python -m pytest tests/test_reference_suite.py tests/test_gpu_parity.py -q -k "reference or scalar or ring or clmul or golden" > gpurun_out/tpc.log 2>&1; echo rc=$? >> gpurun_out/tpc.log
