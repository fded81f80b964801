#!/bin/bash
# Re-create the profiles/rN evidence on a B200 box (run from the repo root,
# e.g. via gpurun).  Each ncu pass runs only after the same command exited 0
# without ncu; outputs land in gpurun_out/ (copy the ones to keep into
# profiles/rN/ and summarise them in profiles/rN/SUMMARY.md).
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python bench.py --steps 5 --warmup 3 --quick --no-cpu > gpurun_out/plain.log 2>&1 &&
ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv \
    --log-file gpurun_out/launch_list_bench.csv \
    python bench.py --steps 5 --warmup 3 --quick --no-cpu > gpurun_out/ncu_ll.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k2_node -s 4 -c 1 \
    -o gpurun_out/k2_node_mul_full \
    python bench.py --steps 5 --warmup 3 --quick --no-cpu > gpurun_out/ncu_full.log 2>&1
python tools/quick_time.py 57637 > gpurun_out/qt57637.log 2>&1 &&
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launch_list_57637.csv \
    python tools/quick_time.py 57637 > gpurun_out/ncu_57637.log 2>&1
python tools/quick_time.py 35851 > gpurun_out/qt35851.log 2>&1 &&
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launch_list_35851.csv \
    python tools/quick_time.py 35851 > gpurun_out/ncu_35851.log 2>&1
python tools/quick_time.py 57637 > /dev/null 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:"toom|k1_|k3_|k4_" -s 7 -c 7 \
    -o gpurun_out/mem57637 python tools/quick_time.py 57637 > gpurun_out/ncu_mem57637.log 2>&1
echo done
