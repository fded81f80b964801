# per-kernel A/B of prebuilt libraries: bash tools/_abk.sh "sizes" dir1 dir2 ...
sizes="$1"; shift
for v in "$@"; do
  cp _old/$v/libf2x.so paper_2201_10473_b200/_build/libf2x.so
  echo "== $v"; timeout 300 python tools/kernel_times.py $sizes 2>&1 | sed 's/void f2x:://g' | tail -40
done
