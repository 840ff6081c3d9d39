O=gpurun_out/r1zi; mkdir -p $O
for F in 2; do echo "FA64=$F"; RF_ATTN_FA64=$F timeout 300 python -m pytest tests/test_gpu_dit.py -x -q -k "reproducible" 2>&1 | tail -1; done > $O/repro.txt
cat $O/repro.txt
