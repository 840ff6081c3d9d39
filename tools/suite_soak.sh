#!/bin/bash
# The full GPU suite N times in fresh processes: a rare hang shows up with the stuck test's
# Python stack (pytest.ini faulthandler_timeout), the GPU's utilisation while stuck and
# the kernel-side wait channel of every thread of the hung process.
N=${1:-3}
LIMIT=${2:-300}
TESTS=${3:-tests}
mkdir -p gpurun_out/soak
for i in $(seq 1 $N); do
  python -m pytest $TESTS -m gpu -x -q > gpurun_out/soak/run$i.log 2>&1 &
  PID=$!
  t=0
  while kill -0 $PID 2>/dev/null && [ $t -lt $LIMIT ]; do sleep 5; t=$((t+5)); done
  if kill -0 $PID 2>/dev/null; then
    echo "run $i HUNG after ${t}s"
    for k in 1 2 3; do nvidia-smi --query-gpu=utilization.gpu,utilization.memory,memory.used,clocks.sm,power.draw --format=csv,noheader; sleep 1; done
    for tdir in /proc/$PID/task/*; do echo "$(basename $tdir) $(cat $tdir/comm) wchan=$(cat $tdir/wchan) $(cat $tdir/syscall 2>/dev/null | cut -d' ' -f1-3)"; done | head -40
    timeout -s KILL 90 /usr/local/cuda/bin/cuda-gdb -batch -p $PID -ex "thread apply all bt 12" > gpurun_out/soak/gdb$i.txt 2>&1
    grep -E "^#|^Thread" gpurun_out/soak/gdb$i.txt | grep -v "^#.*in ?? ()" | head -60
    grep -B2 -A8 "Timeout" gpurun_out/soak/run$i.log | head -12
    kill -9 $PID
    break
  fi
  wait $PID
  echo "run $i rc=$? $(tail -1 gpurun_out/soak/run$i.log | cut -c1-120)"
done
