# A/B quick timing of prebuilt libraries: bash tools/_ab_run.sh "sizes" dir1 dir2 ...
sizes="$1"; shift
for r in 1 2; do for v in "$@"; do
  cp _old/$v/libf2x.so paper_2201_10473_b200/_build/libf2x.so
  echo "== $v"; timeout 300 python tools/quick_time.py $sizes 2>&1 | grep '"kind"' | cut -c1-120
done; done
