O=gpurun_out/r1j; mkdir -p $O
timeout 120 python tools/gemm_trace.py > $O/gemm_trace.txt 2>&1
timeout 300 python -m pytest tests -m gpu -q -x -k "gemm or dit" > $O/pytest.txt 2>&1
timeout 120 python tools/dit_check.py 4 --graph > $O/dit_check.txt 2>&1
grep resid $O/gemm_trace.txt; tail -2 $O/pytest.txt; cat $O/dit_check.txt
