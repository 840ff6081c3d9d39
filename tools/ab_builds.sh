#!/bin/bash
# Usage: build two variants into paper_2605_28657_b200/_lib/libA.so / libB.so (build.build(force=True,
# extra_flags=[...]) + copy), then gpurun -- bash tools/ab_builds.sh
# A/B two builds of the library on one box: alternate copies into the loaded path.
L=paper_2605_28657_b200/_lib
for i in 1 2 3; do
  for v in A B; do
    cp $L/lib$v.so $L/libringflow_b200.so
    echo -n "$v: "; timeout 200 python tools/dit_sustained.py 2>&1 | tail -n 1
  done
done
cp $L/libA.so $L/libringflow_b200.so
