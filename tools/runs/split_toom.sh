# row chunks on forked streams re-measured on the Toom plans (one CUDA graph): F2X_TOOM=2 keeps the depth for < 128-group chunks
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
F2X_TOOM=2 timeout 900 python tools/split_streams.py 17669:4096 35851:4096 17669:16384 --splits 1,2,3,4 2>&1 | grep -v -i warn > gpurun_out/split_toom.log
cat gpurun_out/split_toom.log
