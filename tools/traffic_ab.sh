#!/bin/bash
# DRAM traffic of one DiT forward (ncu, --cache-control none: warm, as in the real forward)
# for _ab_base/ and this tree, then the sustained A/B (tools/ab_dit.sh).
O=gpurun_out/traffic; mkdir -p $O
M="--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --cache-control none -k regex:rf_|gemm -c 700 --csv"
(cd _ab_base && timeout 300 ncu $M --log-file ../$O/base.csv python tools/dit_check.py 4 --no-ref > /dev/null 2>&1)
timeout 300 ncu $M --log-file $O/new.csv python tools/dit_check.py 4 --no-ref > /dev/null 2>&1
for n in base new; do echo "== $n"; python tools/forward_traffic.py $O/$n.csv $O/$n.csv $O/$n.json | tail -4; done
bash tools/ab_dit.sh
