# bench (engine + reference arm) and the d=1024 slicing/unslicing capture -> gpurun_out/
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench.log 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
timeout 600 python bench.py --impl reference --steps 20 --warmup 2 > gpurun_out/bench_ref.log 2>&1; echo "ref rc=$?" >> gpurun_out/bench_ref.log
timeout 900 bash tools/runs/ncu_mem1024.sh > /dev/null 2>&1
