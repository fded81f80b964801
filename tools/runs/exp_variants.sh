# usage: bash tools/runs/exp_variants.sh "RING_SIZES" "FULL_D_SIZES" NAME1 NAME2 ...
# (variants built by tools/build_variant.py; each swapped in for _build/libf2x.so in turn)
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
SIZES=$1; FULL=$2; shift 2
cp paper_2201_10473_b200/_build/libf2x.so /tmp/libf2x_default.so
for v in default "$@"; do
  if [ "$v" = default ]; then cp /tmp/libf2x_default.so paper_2201_10473_b200/_build/libf2x.so
  else cp paper_2201_10473_b200/_build_exp/$v/libf2x.so paper_2201_10473_b200/_build/libf2x.so; fi
  echo "== $v" >> gpurun_out/exp_variants.log
  [ -n "$SIZES" ] && timeout 600 python tools/kernel_times.py $SIZES >> gpurun_out/exp_variants.log 2>&1
  [ -n "$FULL" ] && timeout 600 python tools/kernel_times_full.py $FULL >> gpurun_out/exp_variants.log 2>&1
done
cp /tmp/libf2x_default.so paper_2201_10473_b200/_build/libf2x.so
