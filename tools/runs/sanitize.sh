# usage (one tool per gpurun call): bash tools/runs/sanitize.sh racecheck|memcheck|initcheck|synccheck
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
T=$1
python tools/sanitize_case.py ring 12323 64 > gpurun_out/san_plain.log 2>&1 || exit 1
timeout 1500 compute-sanitizer --tool $T --print-limit 50 python tools/sanitize_case.py ring 12323 64 > gpurun_out/san_${T}_12323.log 2>&1; echo "rc=$?" >> gpurun_out/san_${T}_12323.log
F2X_TOOM=3 timeout 1500 compute-sanitizer --tool $T --print-limit 50 python tools/sanitize_case.py ring 57637 40 > gpurun_out/san_${T}_57637_toom3.log 2>&1; echo "rc=$?" >> gpurun_out/san_${T}_57637_toom3.log
F2X_TOOM=3 F2X_TOOM_SEQ=1 timeout 1500 compute-sanitizer --tool $T --print-limit 50 python tools/sanitize_case.py ring 57637 40 > gpurun_out/san_${T}_57637_toom3_seq.log 2>&1; echo "rc=$?" >> gpurun_out/san_${T}_57637_toom3_seq.log
