O=gpurun_out/r1zp; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke exit $?" >> $O/smoke.log
timeout 600 python bench.py > $O/bench.json 2> $O/bench.err
tail -n 3 $O/pytest_gpu.log $O/smoke.log; python -c "
import json; d=json.load(open('$O/bench.json')); print(d['value'], d['ms_per_step'], d['phase_ms'], d['roofline']['frac'], d['e2e']['value'], d['clocks'], d['toy_path']['value'], d['cpu_baseline']['value'])"
tail -n 3 $O/bench.err
