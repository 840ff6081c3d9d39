#!/bin/bash
# One GPU-box pass: gpu tests, smoke, bench (1 GPU), DiT-forward launch list with DRAM bytes.
# Usage (from this container): gpurun --timeout 1500 -- 'bash tools/gpu_check.sh TAG'
TAG=${1:-run}
O=gpurun_out/$TAG
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/gpu.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke exit $?" >> $O/smoke.log
timeout 600 python bench.py > $O/bench.json 2> $O/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  -k regex:'rf_|gemm' -c 700 --csv --log-file $O/dit_launches.csv python tools/dit_check.py 4 --no-ref > $O/ncu_dit.log 2>&1
tail -n 3 $O/pytest_gpu.log $O/smoke.log; cat $O/bench.json; tail -3 $O/bench.err
