#!/bin/bash
# Profiles for the round's evidence (profiles/): ncu --set full of the DiT forward's top
# kernels (one launch each, mid-forward), and the forward's DRAM traffic launch lists
# (cold: ncu flushes caches before each kernel; warm: --cache-control none).
# Usage: gpurun --timeout 1500 -- 'bash tools/profile_round.sh TAG'
TAG=${1:-prof}
O=gpurun_out/$TAG
mkdir -p $O
P='python tools/dit_check.py 4 --no-ref'
for spec in "gateup:rf_gemm_kernel<\(int\)256, \(int\)3, \(int\)2" "down:rf_gemm_kernel<\(int\)128, \(int\)2, \(int\)2, \(int\)32" \
            "oproj:rf_gemm_kernel<\(int\)128, \(int\)2, \(int\)2, \(int\)128" "qkv:rf_gemm_kernel<\(int\)256, \(int\)5, \(int\)2" \
            "xq_xattn:rf_gemm_kernel<\(int\)128, \(int\)6" "attn_self:rf_attn_fa64_kernel" "norm:rf_dit_norm_mod" \
            "tick_solve:rf_tick_fast_kernel" "decode:rf_decode_tc_kernel" \
            "proj_wide_c5:rf_gemm_kernel<\(int\)256, \(int\)2, \(int\)2"; do
  n=${spec%%:*}; r=${spec#*:}
  if [ $n = tick_solve ]; then prog='python tools/toy_ticks.py 40'; elif [ $n = decode ]; then prog="python tools/decode_one.py 1500 1425 1500 4"
  elif [ $n = proj_wide_c5 ]; then prog="$P --frames=6000"; else prog=$P; fi
  skip=12; if [ $n = decode ]; then skip=2; fi
  timeout 300 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k "regex:$r" -s $skip -c 1 -o $O/$n $prog > $O/$n.log 2>&1
done
M="--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:rf_|gemm -c 700 --csv"
timeout 300 ncu $M --log-file $O/cold.csv $P > /dev/null 2>&1
timeout 300 ncu $M --cache-control none --log-file $O/warm.csv $P > /dev/null 2>&1
ls -la $O
python tools/forward_traffic.py $O/cold.csv $O/warm.csv $O/traffic.json > /dev/null 2>&1
for f in $O/*.ncu-rep; do python tools/ncu_hot.py $f 12 > ${f%.ncu-rep}.hot.txt 2>&1; done
