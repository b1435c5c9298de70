O=gpurun_out/chk2; mkdir -p $O
python -m pytest tests -m gpu -q > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
NKB_LIB=paper_2312_09888_b200/lib/libnekb200_checked.so python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_checked.log 2>&1; echo "pytest(checked) rc=$?" >> $O/pytest_checked.log
bash tools/gpu/c5sweep.sh
tail -n 3 $O/pytest.log $O/pytest_checked.log
