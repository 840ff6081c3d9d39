#!/bin/bash
# A/B an environment switch on one box: sustained DiT forward, alternating, 3 rounds.
# Usage: gpurun -- bash tools/ab_env.sh "VAR=VALUE [VAR2=VALUE2]"
for i in 1 2 3; do
  echo -n "default: "; timeout 200 python tools/dit_sustained.py 2>&1 | tail -n 1
  echo -n "$1: "; timeout 200 env $1 python tools/dit_sustained.py 2>&1 | tail -n 1
done
