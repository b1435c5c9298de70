O=gpurun_out/pre2t; rm -rf $O; mkdir -p $O
python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -m gpu -q -x > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log; tail -n 2 $O/pytest.log
NKB_LIB=paper_2312_09888_b200/lib/libnekb200_checked.so python -m pytest tests/test_gpu_parity.py -m gpu -q -x > $O/pytest_checked.log 2>&1; echo "checked rc=$?" >> $O/pytest_checked.log; tail -n 2 $O/pytest_checked.log
