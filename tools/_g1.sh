O=gpurun_out/r1zm; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_dit.py tests/test_gpu_gemm.py -x -q > $O/pytest.txt 2>&1
tail -2 $O/pytest.txt
timeout 120 python tools/dit_check.py 4 > $O/check.txt 2>&1; head -1 $O/check.txt
RF_DIT_FUSE_NORM=0 timeout 120 python tools/dit_check.py 4 > $O/check0.txt 2>&1; head -1 $O/check0.txt
timeout 1200 python tools/ab.py "RF_DIT_FUSE_NORM=1" "RF_DIT_FUSE_NORM=0" --rounds=5 > $O/ab.txt 2>&1
cat $O/ab.txt
