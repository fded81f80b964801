#!/bin/bash
# A/B/... node-kernel timing of prebuilt libraries (development aid):
#   tools/abn.sh "17669 35851" _old/a _old/b _old/c
sizes="$1"; shift
for r in 1 2; do
  for v in "$@"; do
    cp "$v/libf2x.so" paper_2201_10473_b200/_build/libf2x.so
    echo "== $v"; python tools/kernel_times.py $sizes | sed 's/void f2x:://g'
  done
done
