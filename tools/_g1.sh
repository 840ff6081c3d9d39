O=gpurun_out/r1zb; mkdir -p $O
timeout 120 python tools/attn_bench.py 1:0 2:0 0:0 > $O/attn.txt 2>&1
timeout 60 python tools/attn64_trace.py | tail -4 >> $O/attn.txt 2>&1
timeout 300 python -m pytest tests/test_gpu_dit.py -x -q -k "attention or dit" >> $O/attn.txt 2>&1
cat $O/attn.txt | tail -14
