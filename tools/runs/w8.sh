# experiment: Toom-3 point x = X^w for w != 16 (variant build NAME = w8 / w32, kToomW edited for
# tools/build_variant.py): per-kernel times of the default and the variant, then GPU parity on the variant
# usage: bash tools/runs/w8.sh w8
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out; V=${1:-w8}; rm -f gpurun_out/$V.log
cp paper_2201_10473_b200/_build/libf2x.so /tmp/libf2x_default.so
SIZES="57637:16384 17669 35851 28000 20000 24000 12323:4096"
for lib in default $V; do
  [ $lib = default ] || cp paper_2201_10473_b200/_build_exp/$V/libf2x.so paper_2201_10473_b200/_build/libf2x.so
  echo "== $lib" >> gpurun_out/$V.log
  timeout 600 python tools/kernel_times.py $SIZES 2>&1 | grep "^n=" | cut -c1-330 >> gpurun_out/$V.log
  timeout 600 python tools/kernel_times_full.py 32768 65536 2>&1 | grep "^d=" | cut -c1-330 >> gpurun_out/$V.log
done
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_baseline_batches.py -q 2>&1 | tail -n 6 >> gpurun_out/$V.log
cp /tmp/libf2x_default.so paper_2201_10473_b200/_build/libf2x.so
