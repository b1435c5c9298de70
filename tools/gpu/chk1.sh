# GPU suite on the product library, then the whole suite again on the checked build; bench default
O=gpurun_out/chk1; mkdir -p $O
python -m pytest tests -m gpu -q > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
NKB_LIB=paper_2312_09888_b200/lib/libnekb200_checked.so python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_checked.log 2>&1; echo "pytest(checked) rc=$?" >> $O/pytest_checked.log
python bench.py --steps 20 --warmup 5 --csv $O/csv > $O/bench.json 2> $O/bench.err; echo "bench rc=$?"
python bench.py --config c4 --steps 10 --warmup 3 > $O/bench_c4.json 2> $O/bench_c4.err; echo "bench c4 rc=$?"
python bench.py --config c3 --steps 10 --warmup 3 > $O/bench_c3.json 2> $O/bench_c3.err; echo "bench c3 rc=$?"
python bench.py --config c1 --steps 20 --warmup 5 > $O/bench_c1.json 2> $O/bench_c1.err; echo "bench c1 rc=$?"
tail -2 $O/pytest.log $O/pytest_checked.log
