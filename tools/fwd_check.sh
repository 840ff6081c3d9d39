#!/bin/bash
# One GPU pass for a DiT-forward change: GEMM + DiT GPU tests (incl. the trajectory parity),
# forward accuracy/time, sustained forward rate, per-kernel launch list of one forward (ncu,
# cold, serialised).
# Usage: gpurun --timeout 900 -- 'bash tools/fwd_check.sh TAG'
TAG=${1:-fwd}
O=gpurun_out/$TAG
mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_dit.py tests/test_gpu_dit_trajectory.py -x -q > $O/pytest.log 2>&1; echo "pytest exit $?" >> $O/pytest.log
timeout 200 python tools/dit_check.py 4 > $O/dit_check.txt 2>&1
timeout 200 python tools/dit_sustained.py >> $O/dit_check.txt 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'rf_|gemm' -c 700 --csv \
  --log-file $O/launches.csv python tools/dit_check.py 4 --no-ref > $O/ncu.log 2>&1
python tools/launch_summary.py $O/launches.csv 231 > $O/launch_summary.txt 2>&1
tail -n 15 $O/pytest.log; cat $O/dit_check.txt $O/launch_summary.txt
