O=gpurun_out/r1ze; mkdir -p $O
timeout 300 python -m pytest tests/test_gpu_dit.py -x -q -k "deterministic or reproducible" > $O/neg.txt 2>&1
tail -3 $O/neg.txt
