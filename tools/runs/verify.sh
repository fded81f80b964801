# state check after a restore: smoke, GPU tests, bench -> gpurun_out/
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 2000 python -m pytest tests -m gpu -q -rfEs > gpurun_out/gputest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gputest.log
timeout 900 python bench.py > gpurun_out/bench.log 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
timeout 300 python tools/kernel_times.py 17669 35851 57637:16384 12323:256 > gpurun_out/ktimes.log 2>&1
tail -n 3 gpurun_out/smoke.log gpurun_out/gputest.log gpurun_out/bench.err
