#!/bin/bash
# A/B of the sustained DiT forward on one box: _ab_base/ (a built copy of the previous commit,
# git-ignored) vs this tree, alternating 3 times.
for i in 1 2 3; do
  echo -n "base: "; (cd _ab_base && timeout 120 python tools/dit_sustained.py)
  echo -n "new:  "; timeout 120 python tools/dit_sustained.py
done
