#!/bin/bash
# A/B node-kernel timing of two prebuilt libraries (development aid):
#   tools/ab.sh _old/base _old/perm "17669 35851 57637:16384"
for r in 1 2 3; do
  for v in "$1" "$2"; do
    cp "$v/libf2x.so" paper_2201_10473_b200/_build/libf2x.so
    echo "== $v"; python tools/kernel_times.py $3 | sed 's/void f2x:://g'
  done
done
