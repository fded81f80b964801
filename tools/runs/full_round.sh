cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 2000 python -m pytest tests -m gpu -q -rfEs > gpurun_out/gputest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gputest.log
timeout 900 python bench.py > gpurun_out/bench.log 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
timeout 1500 bash tools/reproduce_profiles.sh > gpurun_out/profiles.log 2>&1
