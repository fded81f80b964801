cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
for v in 2 1 2 1; do
  echo "== F2X_EVAL_LEVELS=$v" >> gpurun_out/el_ab.log
  F2X_EVAL_LEVELS=$v timeout 600 python tools/split_streams.py 17669:4096 --splits 1 --reps 100 >> gpurun_out/el_ab.log 2>&1
done
F2X_EVAL_LEVELS=1 timeout 300 python tools/kernel_times.py 17669 >> gpurun_out/el_ab.log 2>&1
