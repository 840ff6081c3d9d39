O=gpurun_out/r1za; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_codec.py tests/test_decode_gate.py -x -q > $O/pytest.log 2>&1; echo "pytest exit $?" >> $O/pytest.log
tail -n 4 $O/pytest.log
