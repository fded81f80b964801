cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python tools/ct_probe.py 400 0xC9 > gpurun_out/ctprobe.log 2>&1
python tools/ct_probe.py 400 0xC7 >> gpurun_out/ctprobe.log 2>&1
nvidia-smi -q -d POWER,CLOCK,PERFORMANCE | head -80 >> gpurun_out/ctprobe.log 2>&1
